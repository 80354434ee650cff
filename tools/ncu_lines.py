"""Top CUDA source lines by warp-stall samples from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys


def main(path, top=30, by="stall"):
    cur = None
    hdr = None
    lines = []
    total = 0.0
    for row in csv.reader(open(path)):
        if not row:
            continue
        if row[0] == "File Path":
            cur = row[1].split("/")[-1]
            continue
        if row[0] == "Line No":
            hdr = {k: i for i, k in enumerate(row)}
            continue
        if hdr and row[0].isdigit():
            f = lambda v: float(v) if v not in ("", "-") else 0.0
            try:
                s = f(row[4])
                n = f(row[7])
            except ValueError:
                continue
            total += s
            lines.append((s, n, cur, int(row[0]), row[1].strip()[:90]))
    if by == "inst":
        lines.sort(key=lambda x: -x[1])
    else:
        lines.sort(reverse=True)
    print(f"total stall samples {total:.0f}  total instructions {sum(x[1] for x in lines) / 1e6:.1f}M  (sorted by {by})")
    for s, n, f, ln, src in lines[:top]:
        print(f"{100 * s / total:5.1f}% {n / 1e6:8.2f}M  {f}:{ln:<5d} {src}")


if __name__ == "__main__":
    main(sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30, sys.argv[3] if len(sys.argv) > 3 else "stall")
