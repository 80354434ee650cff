"""Write profiles/traffic.json from ncu captures of ONE launch each, beside the algorithmic bytes of that
same launch (so ncu DRAM traffic and the algorithmic figure compare like with like).

    python tools/traffic_update.py key=path.ncu-rep:objective:iteration[:T] ...   (on the GPU box)

key names the bench line (c4:<objective> candidates, c4eval:<objective> evaluation); iteration is the
0-based loop index of the captured launch (tools/prof_split.py: -s 3 -> iteration 3 of T = 100).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def raw_metrics(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, units, vals = rows[0], rows[1], rows[2]

    def get(name):
        i = h.index(name)
        v = float(vals[i].replace(",", ""))
        u = units[i]
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6, "GB": 1e9,
                 "nsecond": 1, "usecond": 1e3, "msecond": 1e6, "second": 1e9, "ns": 1, "us": 1e3, "ms": 1e6,
                 "s": 1e9, "%": 1, "": 1}
        if u not in scale:
            raise ValueError(f"unknown ncu unit {u!r} for {name}")
        return v * scale[u]

    d = {"dram_bytes": get("dram__bytes_read.sum") + get("dram__bytes_write.sum"),
         "duration_ns": get("gpu__time_duration.sum")}
    try:
        d["dmma_pipe_active_pct"] = get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active")
    except ValueError:
        pass
    return d


def algorithmic_bytes(objective, t, T, ps=1_000_000, dim=100, seed=0):
    import torch

    import bench
    from paper_2510_14982_b200 import _lib
    from paper_2510_14982_b200.core import iteration_scalars

    in_dr = torch.empty(ps, dtype=torch.uint8, device="cuda")
    _lib.check(_lib.load().apo_select_dr(seed, t + 1, ps, 0.1, _lib.ptr(in_dr), None, _lib.stream_handle()))
    p_auto = bench.op_mix(seed, t + 1, ps, iteration_scalars(t, T)[0], in_dr.cpu().numpy().astype(bool))
    return ps * bench.bytes_per_eval(dim, p_auto), p_auto


def main(specs):
    path_out = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        doc = json.load(open(path_out))
    except Exception:
        doc = {}
    launches = doc.get("launches", {})
    for spec in specs:
        key, rest = spec.split("=", 1)
        parts = rest.split(":")
        rep, objective, t = parts[0], parts[1], int(parts[2])
        T = int(parts[3]) if len(parts) > 3 else 100
        m = raw_metrics(rep)
        entry = {**m, "launch": f"{objective} ps=1e6 D=100 iteration {t} of T={T} (seed 0)", "report": os.path.basename(rep)}
        if key.startswith("c4:"):  # the candidate / update kernel: the algorithmic bytes of this launch
            entry["algorithmic_bytes"], entry["p_auto"] = algorithmic_bytes(objective, t, T)
            entry["traffic_over_algorithmic"] = round(entry["dram_bytes"] / entry["algorithmic_bytes"], 4)
            entry["algorithmic_gbs"] = round(entry["algorithmic_bytes"] / entry["duration_ns"], 1)
        launches[key] = entry
    doc = {"_source": "ncu --set full, one launch each (tools/traffic_update.py): dram__bytes_read.sum + "
                      "dram__bytes_write.sum, sm__pipe_tensor_subpipe_dmma_cycles_active; algorithmic bytes of the "
                      "same launch from SURVEY 8(d)'s B_eval with that iteration's exact op mix",
           "launches": launches}
    json.dump(doc, open(path_out, "w"), indent=1)
    print(json.dumps(doc, indent=1))


if __name__ == "__main__":
    main(sys.argv[1:])
