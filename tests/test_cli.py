"""The command-line front end keeps the reference's record schema (cli.py:43-77) and exit codes."""

import json
import os

import numpy as np
import pytest

from paper_2510_14982_b200 import cli


def test_format_number_matches_reference_rules():
    assert cli.format_number(0.0) == "0"
    assert cli.format_number(float("nan")) == "nan"
    assert cli.format_number(float("-inf")) == "-inf"
    assert cli.format_number(430 / 64) == "6.71875"
    assert cli.format_number(1234567.0) == "1.23457E+06"
    assert cli.format_number(0.000123456789) == "1.23457E-04"
    assert cli.format_number(-2500.0) == "-2500"


def _records(tmp_path):
    rows = [("sphere", "sequential", 430.0, 1.0), ("sphere", "parallel", 64.0, 1.0),
            ("rosenbrock", "sequential", 211.0, 3.0), ("rosenbrock", "parallel", 35.0, 3.5)]
    path = tmp_path / "bench.csv"
    text = ",".join(cli.BENCH_COLUMNS) + "\n"
    for fn, mode, secs, fit in rows:
        text += f"{fn},100,10,50,5,0,{mode},1,{fit},{secs}\n"
    path.write_text(text)
    return path


def test_report_joins_modes_into_speedups(tmp_path, capsys):
    """Criterion 7 of the reference's acceptance suite: 430/64 -> 6.72 and 211/35 -> 6.03."""
    path = _records(tmp_path)
    assert cli.main(["report", "--in", str(path), "--format", "csv"]) == 0
    out = capsys.readouterr().out.splitlines()
    assert out[0].split(",") == list(cli.REPORT_COLUMNS)
    speed = {line.split(",")[0]: line.split(",")[-1] for line in out[1:]}
    assert speed == {"rosenbrock": "6.03", "sphere": "6.72"}
    assert cli.main(["report", "--in", str(path)]) == 0
    assert "| 2 | sphere | 100 |" in capsys.readouterr().out


def test_report_rejects_bad_records_and_writes_atomically(tmp_path):
    bad = tmp_path / "bad.csv"
    bad.write_text("function,ps\nsphere,1\n")
    assert cli.main(["report", "--in", str(bad)]) == 2
    out = tmp_path / "table.md"
    assert cli.main(["report", "--in", str(_records(tmp_path)), "--out", str(out)]) == 0
    assert out.read_text().startswith("| No. |") and not [p for p in os.listdir(tmp_path) if p.startswith(".partial")]


def test_seed_resolution(monkeypatch):
    monkeypatch.delenv("PROTOZOA_SEED", raising=False)
    assert cli.resolve_seed(None) == 0 and cli.resolve_seed(7) == 7
    monkeypatch.setenv("PROTOZOA_SEED", "42")
    assert cli.resolve_seed(None) == 42 and cli.resolve_seed(3) == 3
    monkeypatch.setenv("PROTOZOA_SEED", "x")
    with pytest.raises(ValueError):
        cli.resolve_seed(None)


def test_pgm_reader(tmp_path):
    img = (np.arange(12, dtype=np.uint8) * 20).reshape(3, 4)
    p = tmp_path / "a.pgm"
    p.write_bytes(b"P5\n# comment\n4 3\n255\n" + img.tobytes())
    assert np.array_equal(cli.read_image(p), img)
    q = tmp_path / "b.pgm"
    q.write_bytes(b"P2\n4 3\n254\n" + b"0 " * 12)
    assert cli.main(["threshold", "--image", str(q)]) == 4


@pytest.mark.gpu
def test_bench_and_threshold_commands(tmp_path, capsys):
    out = tmp_path / "b.csv"
    assert cli.main(["bench", "--function", "cec2022_f1", "--ps", "64", "--dim", "10", "--iters", "20",
                     "--runs", "2", "--out", str(out)]) == 0
    lines = out.read_text().splitlines()
    assert lines[0].split(",") == list(cli.BENCH_COLUMNS) and len(lines) == 3
    runs = (tmp_path / "b_runs.csv").read_text().splitlines()
    assert runs[0].split(",") == list(cli.RUN_COLUMNS) and len(runs) == 5
    assert cli.main(["bench", "--function", "sphere", "--ps", "32", "--dim", "4", "--iters", "5", "--runs", "1",
                     "--format", "json"]) == 0
    rec = json.loads(capsys.readouterr().out)["records"]
    assert {r["mode"] for r in rec} == {"sequential", "parallel"}
    rnd = np.random.default_rng(0)
    img = np.clip(np.where(rnd.random((128, 128)) < 0.5, rnd.normal(60, 10, (128, 128)),
                           rnd.normal(180, 12, (128, 128))), 0, 255).astype(np.uint8)
    np.save(tmp_path / "img.npy", img)
    assert cli.main(["threshold", "--image", str(tmp_path / "img.npy"), "--levels", "2", "--method", "kapur"]) == 0
    assert capsys.readouterr().out.startswith("thresholds=")


def _strip_seconds(lines):
    import re

    return [re.sub(r"(seconds=|Avg\. Time \(s\) )\S+", r"\1<t>", ln) for ln in lines]


@pytest.mark.gpu
def test_threshold_command_matches_reference_cli(tmp_path, capsys):
    """`threshold --runs --engine both --check-oracle --emit` prints the reference CLI's lines
    (cli.py:262-303: per-run seed/threshold/variance, per-mode averages, the oracle check) and writes the
    same binarised PGM; only the seconds differ.  The reference (baseline/_ref, numba) runs beside it."""
    import sys

    ref_site = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_site, "protozoa")):
        pytest.skip("reference not installed in baseline/_ref")
    rnd = np.random.default_rng(3)
    img = np.clip(np.where(rnd.random((96, 80)) < 0.4, rnd.normal(70, 12, (96, 80)),
                           rnd.normal(190, 14, (96, 80))), 0, 255).astype(np.uint8)
    pgm = tmp_path / "img.pgm"
    pgm.write_bytes(b"P5\n80 96\n255\n" + img.tobytes())
    args = ["threshold", "--image", str(pgm), "--runs", "3", "--engine", "both", "--seed", "5", "--check-oracle",
            "--emit-format", "p2"]
    assert cli.main(args + ["--emit", str(tmp_path / "ours.pgm")]) == 0
    ours = capsys.readouterr().out.splitlines()
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_cli")
    sys.path.insert(0, ref_site)
    try:
        from protozoa import cli as ref_cli
    finally:
        sys.path.remove(ref_site)
    assert ref_cli.main(args + ["--emit", str(tmp_path / "ref.pgm")]) == 0
    ref = capsys.readouterr().out.splitlines()
    assert _strip_seconds(ours) == _strip_seconds(ref)
    assert (tmp_path / "ours.pgm").read_bytes() == (tmp_path / "ref.pgm").read_bytes()


@pytest.mark.gpu
def test_bench_command_records_match_reference_cli(tmp_path):
    """`bench --format json` writes the reference CLI's records (cli.py:166-257): same functions, sizes,
    seeds, modes and per-run best fitness bit for bit (both modes run the bit-exact keyed stream); only
    seconds and the worker count (CPU threads there, GPUs here) differ."""
    import sys

    ref_site = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_site, "protozoa")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_cli")
    sys.path.insert(0, ref_site)
    try:
        from protozoa import cli as ref_cli
    finally:
        sys.path.remove(ref_site)
    args = ["bench", "--function", "rosenbrock", "--ps", "48", "--dim", "6", "--iters", "30", "--runs", "3",
            "--seed", "11", "--engine", "both", "--format", "json"]
    assert cli.main(args + ["--out", str(tmp_path / "ours.json")]) == 0
    assert ref_cli.main(args + ["--out", str(tmp_path / "ref.json")]) == 0
    ours = json.loads((tmp_path / "ours.json").read_text())["records"]
    ref = json.loads((tmp_path / "ref.json").read_text())["records"]

    def strip(recs):
        out = []
        for r in recs:
            r = {k: v for k, v in r.items() if k not in ("avg_seconds", "workers")}
            r["per_run"] = [{k: v for k, v in p.items() if k != "seconds"} for p in r["per_run"]]
            out.append(r)
        return out

    assert strip(ours) == strip(ref)
