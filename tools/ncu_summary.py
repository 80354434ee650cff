"""Summarise an .ncu-rep: key SOL metrics + instruction mix + stall mix (reads locally, no GPU)."""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "Compute (SM) Throughput", "Registers Per Thread",
        "Achieved Occupancy", "Theoretical Occupancy", "Issued Ipc Active", "Issue Slots Busy", "Executed Instructions",
        "Warp Cycles Per Issued Instruction", "L2 Hit Rate", "L1/TEX Hit Rate", "Eligible Warps Per Scheduler",
        "Avg. Active Threads Per Warp", "Grid Size", "Dynamic Shared Memory Per Block"]


def main(path, top=25):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    res = {}
    for r in rows[1:]:
        d = dict(zip(hdr, r))
        if d.get("Metric Name") in KEYS:
            res[d["Metric Name"]] = d["Metric Value"] + " " + d.get("Metric Unit", "")
    print("kernel:", rows[1][hdr.index("Kernel Name")][:100] if len(rows) > 1 else "?")
    for k in KEYS:
        if k in res:
            print(f"  {k:38s} {res[k]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    h = rr[0]
    for name in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                 "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
                 "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active",
                 "sm__ops_path_tensor_src_fp64.sum.pct_of_peak_sustained_elapsed",
                 "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                 "dram__throughput.avg.pct_of_peak_sustained_elapsed"):
        if name in h:
            print(f"  {name:38s} {rr[2][h.index(name)]} {rr[1][h.index(name)]}")
    sass = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "sass"],
                          capture_output=True, text=True).stdout
    srows = list(csv.reader(io.StringIO(sass)))
    hdr = srows[1]
    ix = {x: i for i, x in enumerate(hdr)}
    ops, stalls = collections.Counter(), collections.Counter()
    tot = st = 0.0
    reasons = collections.Counter()
    for r in srows[2:]:
        if len(r) < len(hdr):
            continue
        src = r[ix["Source"]].strip()
        toks = src.split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        op = op.split(".")[0]
        n = float(r[ix["Instructions Executed"]] or 0)
        s = float(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ops[op] += n
        stalls[op] += s
        tot += n
        st += s
        for k in hdr:
            if k.startswith("stall_") and "Not Issued" not in k:
                try:
                    reasons[k] += float(r[ix[k]] or 0)
                except ValueError:
                    pass
    print(f"  instructions {tot:.4g}  stall samples {st:.4g}")
    for op, n in ops.most_common(top):
        print(f"    {op:10s} {n / 1e6:9.2f}M {100 * n / tot:5.1f}%  stall {100 * stalls[op] / max(st, 1):5.1f}%")
    rs = sum(reasons.values()) or 1
    print("  stall reasons:", ", ".join(f"{k[6:]} {100 * v / rs:.0f}%" for k, v in reasons.most_common(8)))


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 25)
