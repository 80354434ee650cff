"""Per-kernel time share from an ncu --metrics gpu__time_duration.sum --csv launch list."""
import collections
import csv
import sys


def main(path, skip_prefix=("k_init", "k_iota")):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    hdr, rows = rows[0], rows[1:]
    ix = {k: i for i, k in enumerate(hdr)}
    tot = collections.Counter()
    cnt = collections.Counter()
    for r in rows:
        if r[ix["Metric Name"]] != "gpu__time_duration.sum":
            continue
        name = r[ix["Kernel Name"]].split("(")[0].replace("<unnamed>::", "")
        if name.startswith(skip_prefix):
            continue
        tot[name] += float(r[ix["Metric Value"]]) / 1e3
        cnt[name] += 1
    s = sum(tot.values())
    print(f"{'kernel':70s} {'launches':>8s} {'total_us':>10s} {'avg_us':>10s} {'share':>6s}")
    for k, v in tot.most_common():
        print(f"{k[:70]:70s} {cnt[k]:8d} {v:10.1f} {v / cnt[k]:10.1f} {100 * v / s:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
