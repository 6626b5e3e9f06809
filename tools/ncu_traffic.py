"""Summarise ncu passes over one full-pool sweep into
profiles/dp_relax_traffic.json (read by bench.py for roofline.traffic /
achieved / frac):

    # 1) metrics of every relax launch of one D1 pool sweep
    ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,\
lts__t_bytes.sum,l1tex__t_bytes.sum,smsp__inst_executed.sum --clock-control none \
        -k regex:dp_relax --csv --log-file gpurun_out/relax_traffic.csv \
        python tools/profile_dp.py --config D1
    # 2) one --set full capture of a mid-sweep dp_relax_compact launch
    bash tools/gpu/ncu_relax.sh relax_full
    python tools/ncu_traffic.py gpurun_out/relax_traffic.csv D1 1786 gpurun_out/relax_full.ncu-rep

The JSON records the library's hapt_version (the DP kernel generation):
bench.py ignores counters taken on another generation.
"""
import collections
import csv
import io
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "nsecond": 1e-9,
         "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0, "second": 1.0,
         "inst": 1, "": 1, "%": 1, "warp": 1, "cycle": 1}

FULL = {
    "issue_slots_busy_pct": "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "eligible_warps_per_scheduler": "smsp__warps_eligible.avg.per_cycle_active",
    "active_warps_per_scheduler": "smsp__warps_active.avg.per_cycle_active",
    "cycles_per_issued_instruction": "smsp__average_warp_latency_per_inst_issued.ratio",
    "achieved_occupancy_pct": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "dram_bytes": None,
}


def full_stats(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, v = rows[0], rows[2]
    d = {h[i]: v[i] for i in range(len(h))}
    res = {k: float(d[m].replace(",", "")) for k, m in FULL.items() if m and m in d}
    stalls = {k: float(d[k].replace(",", "") or 0) for k in h
              if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls, key=lambda k: -stalls[k])[:4]
    res["stall_share"] = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""):
                          round(stalls[k] / tot, 4) for k in top}
    res["capture"] = os.path.basename(rep)
    return res


def main(path, config, pool, full=None):
    from paper_2509_24859_b200 import _lib

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
        "hapt_version": _lib.load().hapt_version(),
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
    if full:
        out["ncu_full"] = full_stats(full)
    with open(os.path.join(REPO, "profiles", "dp_relax_traffic.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main(*sys.argv[1:])
