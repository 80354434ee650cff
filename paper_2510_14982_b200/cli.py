"""Command-line front end with the reference's record schema.

    python -m paper_2510_14982_b200.cli bench --function cec2022_f6 --ps 100000 --dim 100 --iters 100 --runs 3
    python -m paper_2510_14982_b200.cli report --in bench.csv
    python -m paper_2510_14982_b200.cli threshold --image img.npy --levels 3 --method kapur

The reference CLI (/root/reference/pkg/src/protozoa/cli.py) emits bench
records per engine mode (columns ``cli.py:43-55``), formats numbers with 6
significant digits (``format_number``, ``cli.py:62-77``), writes outputs
atomically and resolves the seed flag > ``PROTOZOA_SEED`` > 0
(``cli.py:122-150``).  This front end keeps those contracts so existing
report tooling reads its output unchanged; the runs themselves go through
this package's device engine.  Exit codes: 0 ok, 2 usage/validation,
3 I/O, 4 image parse failure (``cli.py:466-483``).
"""

from __future__ import annotations

import argparse
import csv
import io
import json
import math
import os
import sys
import tempfile
from typing import List, Optional

BENCH_COLUMNS = ("function", "ps", "dim", "iters", "runs", "seed", "mode", "workers", "avg_best_fit",
                 "avg_seconds")
RUN_COLUMNS = ("function", "ps", "dim", "iters", "mode", "workers", "run_seed", "best_fit", "seconds")
REPORT_COLUMNS = ("function", "ps", "dim", "iters", "seed", "runs", "seq_avg_best_fit", "seq_avg_seconds",
                  "par_avg_best_fit", "par_avg_seconds", "speedup")


class ImageError(ValueError):
    """An image the threshold command cannot read."""


def format_number(value: float) -> str:
    """Six significant digits; scientific below 1e-3 or from 1e6 up; "0", "nan", "inf" spelled out."""
    v = float(value)
    if v == 0.0:
        return "0"
    if v != v:
        return "nan"
    if v in (math.inf, -math.inf):
        return "inf" if v > 0 else "-inf"
    return f"{v:.5E}" if (abs(v) >= 1e6 or abs(v) < 1e-3) else f"{v:.6g}"


def resolve_seed(flag: Optional[int]) -> int:
    if flag is not None:
        return flag
    text = os.environ.get("PROTOZOA_SEED")
    if text is None:
        return 0
    try:
        seed = int(text)
    except ValueError:
        raise ValueError(f"PROTOZOA_SEED must be an integer, got {text!r}") from None
    if not 0 <= seed < 2 ** 64:
        raise ValueError("PROTOZOA_SEED must fit in an unsigned 64-bit word")
    return seed


def atomic_write(path, text) -> None:
    data = text.encode("utf-8") if isinstance(text, str) else text
    folder = os.path.dirname(os.path.abspath(os.fspath(path))) or "."
    fd, tmp = tempfile.mkstemp(dir=folder, prefix=".partial-")
    try:
        with os.fdopen(fd, "wb") as fh:
            fh.write(data)
        os.replace(tmp, path)
    except BaseException:
        try:
            os.unlink(tmp)
        except OSError:
            pass
        raise


def _csv(rows, columns) -> str:
    buf = io.StringIO()
    w = csv.writer(buf, lineterminator="\n")
    w.writerow(columns)
    w.writerows(rows)
    return buf.getvalue()


# ---------------------------------------------------------------------------- bench


def bench_records(result, ps: int, dim: int, iters: int, seed: int) -> List[dict]:
    out = []
    for kind in ("sequential", "parallel"):
        agg = result.per_mode.get(kind)
        if agg is None:
            continue
        out.append({"function": result.objective_name, "ps": ps, "dim": dim, "iters": iters, "runs": result.runs,
                    "seed": seed, "mode": agg.mode, "workers": int(agg.workers),
                    "avg_best_fit": float(agg.avg_best_fitness), "avg_seconds": float(agg.avg_seconds),
                    "per_run": [{"run_seed": seed + k, "best_fit": float(agg.best_fitness[k]),
                                 "seconds": float(agg.seconds[k])} for k in range(result.runs)]})
    return out


def bench_csv(records) -> str:
    return _csv([[r["function"], r["ps"], r["dim"], r["iters"], r["runs"], r["seed"], r["mode"], r["workers"],
                  format_number(r["avg_best_fit"]), format_number(r["avg_seconds"])] for r in records],
                BENCH_COLUMNS)


def runs_csv(records) -> str:
    return _csv([[r["function"], r["ps"], r["dim"], r["iters"], r["mode"], r["workers"], p["run_seed"],
                  format_number(p["best_fit"]), format_number(p["seconds"])]
                 for r in records for p in r["per_run"]], RUN_COLUMNS)


def modes_for(engine: str, workers) -> list:
    """cli.py:153-159: seq and/or par (par with --workers, default "auto")."""
    import paper_2510_14982_b200 as pz

    modes = []
    if engine in ("seq", "both"):
        modes.append(pz.EngineMode.sequential())
    if engine in ("par", "both"):
        modes.append(pz.EngineMode.parallel(workers if workers is not None else "auto"))
    return modes


def cmd_bench(args) -> int:
    import paper_2510_14982_b200 as pz

    seed = resolve_seed(args.seed)
    if not args.lower < args.upper:
        raise ValueError(f"--lower must be below --upper, got [{args.lower}, {args.upper}]")
    cfg = pz.ApoConfig(ps=args.ps, dim=args.dim, bounds=pz.Bounds(args.lower, args.upper, args.dim),
                       max_iterations=args.iters, seed=seed, rng=args.rng)
    modes = modes_for(args.engine, args.workers)
    result = pz.benchmark(cfg, args.function, args.runs, modes=modes)
    records = bench_records(result, args.ps, args.dim, args.iters, seed)
    fmt = args.format or ("json" if args.out and str(args.out).endswith(".json") else "csv")
    if fmt == "json":
        text = json.dumps({"records": records}, indent=2, sort_keys=True) + "\n"
        sys.stdout.write(text) if args.out is None else atomic_write(args.out, text)
    elif args.out is None:
        sys.stdout.write(bench_csv(records))
    else:
        atomic_write(args.out, bench_csv(records))
        stem, ext = os.path.splitext(os.fspath(args.out))
        atomic_write(stem + "_runs" + (ext or ".csv"), runs_csv(records))
    return 0


# ---------------------------------------------------------------------------- report


def load_records(path) -> List[dict]:
    with open(path, encoding="utf-8") as fh:
        text = fh.read()
    if text.lstrip()[:1] in ("{", "["):
        payload = json.loads(text)
        rows = payload.get("records", []) if isinstance(payload, dict) else payload
    else:
        rows = list(csv.DictReader(io.StringIO(text)))
    out = []
    for row in rows:
        try:
            out.append({"function": str(row["function"]), "ps": int(row["ps"]), "dim": int(row["dim"]),
                        "iters": int(row["iters"]), "runs": int(row["runs"]), "seed": int(row["seed"]),
                        "mode": str(row["mode"]), "avg_best_fit": float(row["avg_best_fit"]),
                        "avg_seconds": float(row["avg_seconds"])})
        except (KeyError, TypeError, ValueError) as exc:
            raise ValueError(f"{path}: not a bench record ({exc!r})") from None
    return out


def join_records(records) -> List[dict]:
    groups: dict = {}
    for rec in records:
        key = (rec["function"], rec["ps"], rec["dim"], rec["iters"], rec["seed"])
        if rec["mode"] not in ("sequential", "parallel"):
            raise ValueError(f"unknown mode {rec['mode']!r} for {key}")
        if rec["mode"] in groups.setdefault(key, {}):
            raise ValueError(f"duplicate {rec['mode']} record for {key}")
        groups[key][rec["mode"]] = rec
    rows = []
    for key in sorted(groups):
        pair = groups[key]
        if len(pair) < 2:
            print(f"report: skipping {key}: only a {next(iter(pair))} record", file=sys.stderr)
            continue
        seq, par = pair["sequential"], pair["parallel"]
        if seq["runs"] != par["runs"]:
            raise ValueError(f"run counts differ for {key}: {seq['runs']} vs {par['runs']}")
        rows.append({"function": key[0], "ps": key[1], "dim": key[2], "iters": key[3], "seed": key[4],
                     "runs": seq["runs"], "seq_avg_best_fit": seq["avg_best_fit"],
                     "seq_avg_seconds": seq["avg_seconds"], "par_avg_best_fit": par["avg_best_fit"],
                     "par_avg_seconds": par["avg_seconds"],
                     "speedup": seq["avg_seconds"] / par["avg_seconds"] if par["avg_seconds"] else math.inf})
    return rows


def report_text(rows, fmt: str) -> str:
    if fmt == "csv":
        return _csv([[r["function"], r["ps"], r["dim"], r["iters"], r["seed"], r["runs"],
                      format_number(r["seq_avg_best_fit"]), format_number(r["seq_avg_seconds"]),
                      format_number(r["par_avg_best_fit"]), format_number(r["par_avg_seconds"]),
                      f"{r['speedup']:.2f}"] for r in rows], REPORT_COLUMNS)
    out = ["| No. | Function | PS | Seq Fit | Seq Time | Par Fit | Par Time | Speedup |",
           "| --- | --- | --- | --- | --- | --- | --- | --- |"]
    for n, r in enumerate(rows, 1):
        out.append(f"| {n} | {r['function']} | {r['ps']} | {format_number(r['seq_avg_best_fit'])} | "
                   f"{format_number(r['seq_avg_seconds'])} | {format_number(r['par_avg_best_fit'])} | "
                   f"{format_number(r['par_avg_seconds'])} | {r['speedup']:.2f} |")
    return "\n".join(out) + "\n"


def cmd_report(args) -> int:
    records = [r for path in args.inputs for r in load_records(path)]
    text = report_text(join_records(records), args.format)
    sys.stdout.write(text) if args.out is None else atomic_write(args.out, text)
    return 0


# ---------------------------------------------------------------------------- threshold


def read_image(path) -> "np.ndarray":
    """8-bit grey image from .npy or PGM/PPM (imaging.load_image_file)."""
    import numpy as np

    if str(path).endswith(".npy"):
        img = np.load(path)
        if img.ndim != 2 or img.dtype != np.uint8:
            raise ImageError(f"{path}: expected a 2-D uint8 array")
        return img
    from .imaging import ImageFormatError, load_image_file

    try:
        return load_image_file(path).pixels
    except ImageFormatError as exc:
        raise ImageError(f"{path}: {exc}") from None


def cmd_threshold(args) -> int:
    import paper_2510_14982_b200 as pz

    try:
        img = read_image(args.image)
    except OSError:
        raise
    except ImageError:
        raise
    except Exception as exc:
        raise ImageError(f"{args.image}: {exc}") from None
    seed = resolve_seed(args.seed)
    if not (args.levels == 1 and args.method == "otsu"):  # multilevel: no reference counterpart
        res = pz.apo_multithreshold(img, args.levels, args.method, ps=args.ps, iterations=args.iters, seed=seed)
        print(f"thresholds={','.join(str(t) for t in res.thresholds)} {args.method}={format_number(res.value)}")
        return 0
    # the reference's threshold command (cli.py:262-303): --runs seeds per mode, per-run lines, averages,
    # optional binarised output of the last run and the exhaustive-search oracle check (exit 1 on mismatch)
    from statistics import fmean

    from . import imaging

    gray = pz.GrayImage(img)
    oracle = imaging.brute_force_otsu(imaging.histogram(gray)) if args.check_oracle else None
    mismatches, last = 0, None
    for mode in modes_for(args.engine, args.workers):
        thresholds, seconds = [], []
        for r in range(args.runs):
            res = pz.apo_threshold(gray, ps=args.ps, iterations=args.iters, seed=seed + r, mode=mode)
            thresholds.append(res.threshold)
            seconds.append(res.run.wall_clock_seconds)
            last = res
            print(f"{mode.kind} run {r + 1}: seed={seed + r} threshold={res.threshold} "
                  f"variance={format_number(res.variance)} seconds={format_number(res.run.wall_clock_seconds)}")
            if oracle is not None and res.variance != oracle[1]:
                mismatches += 1
                print(f"oracle mismatch: {mode.kind} run {r + 1} reached {res.variance!r}, "
                      f"exhaustive search reaches {oracle[1]!r} at t={oracle[0]}", file=sys.stderr)
        print(f"{mode.kind} Avg. Best Th. {fmean(thresholds):.2f}  Avg. Time (s) {format_number(fmean(seconds))}")
    if args.emit is not None and last is not None:
        black_white = imaging.apply_threshold(gray, last.threshold)
        atomic_write(args.emit, imaging.write_pgm(black_white, binary=args.emit_format == "p5"))
    if oracle is not None:
        if mismatches:
            return 1
        print(f"oracle check: ok (t={oracle[0]}, variance={format_number(oracle[1])})")
    return 0


# ---------------------------------------------------------------------------- wiring


def _int_at_least(lo):
    def parse(text):
        try:
            v = int(text)
        except ValueError:
            raise argparse.ArgumentTypeError(f"expected an integer, got {text!r}") from None
        if v < lo:
            raise argparse.ArgumentTypeError(f"expected an integer >= {lo}, got {v}")
        return v

    return parse


def _workers(text):
    """cli.py:110-119: a worker count >= 1 or "auto"."""
    if text == "auto":
        return "auto"
    try:
        v = int(text)
    except ValueError:
        raise argparse.ArgumentTypeError(f"expected a worker count or 'auto', got {text!r}") from None
    if v < 1:
        raise argparse.ArgumentTypeError(f"worker count must be >= 1, got {v}")
    return v


def _seed(text):
    v = _int_at_least(0)(text)
    if v >= 2 ** 64:
        raise argparse.ArgumentTypeError("seed must fit in an unsigned 64-bit word")
    return v


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="paper_2510_14982_b200", description=__doc__.splitlines()[0])
    sub = p.add_subparsers(dest="command", required=True)
    b = sub.add_parser("bench", help="run one objective across seeds and engine modes")
    b.add_argument("--function", required=True, help="reference name (sphere, ...) or cec2022_f1..12")
    b.add_argument("--ps", type=_int_at_least(1), default=1000)
    b.add_argument("--dim", type=_int_at_least(1), default=1000)
    b.add_argument("--iters", type=_int_at_least(0), default=1000)
    b.add_argument("--runs", type=_int_at_least(1), default=5)
    b.add_argument("--seed", type=_seed, default=None)
    b.add_argument("--engine", choices=("seq", "par", "both"), default="both")
    b.add_argument("--workers", type=_workers, default=None)
    b.add_argument("--rng", choices=("keyed", "philox"), default="keyed")
    b.add_argument("--lower", type=float, default=-100.0)
    b.add_argument("--upper", type=float, default=100.0)
    b.add_argument("--out", default=None)
    b.add_argument("--format", choices=("csv", "json"), default=None)
    b.set_defaults(handler=cmd_bench)
    t = sub.add_parser("threshold", help="multilevel Otsu / Kapur thresholds of an image")
    t.add_argument("--image", required=True, help=".npy (uint8 2-D) or PGM/PPM (P2/P3/P5/P6)")
    t.add_argument("--levels", type=_int_at_least(1), default=1)
    t.add_argument("--method", choices=("otsu", "kapur"), default="otsu")
    t.add_argument("--ps", type=_int_at_least(1), default=100)
    t.add_argument("--iters", type=_int_at_least(0), default=50)
    t.add_argument("--seed", type=_seed, default=None)
    t.add_argument("--runs", type=_int_at_least(1), default=5)
    t.add_argument("--engine", choices=("seq", "par", "both"), default="seq")
    t.add_argument("--workers", type=_workers, default=None)
    t.add_argument("--emit", default=None, help="write the binarized last run here")
    t.add_argument("--emit-format", choices=("p5", "p2"), default="p5")
    t.add_argument("--check-oracle", action="store_true",
                   help="compare every run with the exhaustive search; exit 1 on a mismatch")
    t.set_defaults(handler=cmd_threshold)
    r = sub.add_parser("report", help="join sequential/parallel bench records into a speedup table")
    r.add_argument("--in", dest="inputs", nargs="+", required=True)
    r.add_argument("--format", choices=("markdown", "csv"), default="markdown")
    r.add_argument("--out", default=None)
    r.set_defaults(handler=cmd_report)
    return p


def main(argv: Optional[List[str]] = None) -> int:
    args = build_parser().parse_args(argv)
    try:
        return args.handler(args)
    except ImageError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 4
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2
    except OSError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 3


if __name__ == "__main__":
    sys.exit(main())
