"""Summarise an ncu metrics pass over one full-pool sweep into
profiles/dp_relax_traffic.json (read by bench.py for roofline.traffic).

    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_bytes.sum,l1tex__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
        -k regex:dp_relax --csv --log-file gpurun_out/relax_traffic.csv \
        python tools/profile_dp.py --config D1
    python tools/ncu_traffic.py gpurun_out/relax_traffic.csv D1 1786 [label]
"""
import collections
import csv
import json
import os
import sys

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
         "inst": 1, "": 1}


def main(path, config, pool, label="dp_relax"):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ii, mi, vi, ui = (h.index(x) for x in ("ID", "Metric Name", "Metric Value", "Metric Unit"))
    per = collections.defaultdict(dict)
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        per[r[ii]][r[mi]] = float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1.0)
    n = len(per)
    tot = collections.Counter()
    for d in per.values():
        tot.update(d)
    out = {
        "kernel": label,
        "config": config,
        "pool_candidates": int(pool),
        "launches": n,
        "dram_bytes_per_launch": (tot["dram__bytes_read.sum"] + tot["dram__bytes_write.sum"]) / n,
        "dram_read_bytes_per_launch": tot["dram__bytes_read.sum"] / n,
        "dram_write_bytes_per_launch": tot["dram__bytes_write.sum"] / n,
        "l2_bytes_per_launch": tot["lts__t_bytes.sum"] / n,
        "l1_bytes_per_launch": tot["l1tex__t_bytes.sum"] / n,
        "instructions_per_launch": tot["smsp__inst_executed.sum"] / n,
        "mean_duration_s_serialised_cold": tot["gpu__time_duration.sum"] / n,
        "source": os.path.basename(path),
    }
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    with open(os.path.join(repo, "profiles", "dp_relax_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
