"""Per-kernel share of an ncu launch list (gpu__time_duration.sum, --csv).

    python tools/kernel_share.py gpurun_out/launches.csv
"""
import collections
import csv
import sys


def main(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    t, n = collections.Counter(), collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) > vi:
            name = r[ki].split("(")[0].replace("hapt::<unnamed>::", "")
            t[name] += float(r[vi].replace(",", ""))
            n[name] += 1
    tot = sum(t.values())
    print(f"total {tot / 1e3:.1f} us over {sum(n.values())} launches")
    for k, v in t.most_common(12):
        print(f"{k[:60]:60s} {n[k]:5d} {v / 1e3:9.1f} us {100 * v / tot:5.1f}%")


if __name__ == "__main__":
    main(sys.argv[1])
