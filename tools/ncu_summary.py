"""Summary of one ncu --set full capture (one kernel launch): key SOL /
scheduler / memory counters, stall reasons and the SASS basic blocks that
take the most instructions.

    python tools/ncu_summary.py gpurun_out/x.ncu-rep [n_blocks]
"""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "lts__t_bytes.sum", "l1tex__t_bytes.sum", "smsp__inst_executed.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__warps_active.avg.per_cycle_active",
        "smsp__average_warp_latency_per_inst_issued.ratio",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size"]


def ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def main(rep, nblocks=25):
    rows = list(csv.reader(io.StringIO(ncu(rep, "--page", "raw", "--csv"))))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i], u[i]) for i in range(len(h))}
    for k in KEYS:
        if k in d:
            print(f"{k:60s} {d[k][0]:>18s} {d[k][1]}")
    keys = [k for k in h if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    val = {k: float(d[k][0].replace(",", "") or 0) for k in keys}
    tot = sum(val.values()) or 1
    print("stall reasons (share of samples):")
    for k in sorted(keys, key=lambda x: -val[x])[:8]:
        print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):30s} {100 * val[k] / tot:5.1f}%")
    src = list(csv.reader(io.StringIO(ncu(rep, "--page", "source", "--csv", "--print-source",
                                          "sass"))))
    hh = src[1]
    isrc, iss = hh.index("Source"), hh.index("Warp Stall Sampling (All Samples)")
    iex = hh.index("Instructions Executed")
    data = src[2:]
    tex = sum(float(r[iex] or 0) for r in data) or 1
    tss = sum(float(r[iss] or 0) for r in data) or 1
    blocks, cur = [], None
    for n, r in enumerate(data):
        ex = float(r[iex] or 0)
        if cur is None or ex != cur["ex"]:
            cur = {"start": n, "ex": ex, "n": 0, "ss": 0.0, "first": r[isrc].strip()}
            blocks.append(cur)
        cur["n"] += 1
        cur["ss"] += float(r[iss] or 0)
        cur["end"] = n
    print(f"SASS blocks (warp instructions {tex:.0f}; [first-last] executions x length):")
    for b in sorted(blocks, key=lambda b: -b["ex"] * b["n"])[:int(nblocks)]:
        print(f"  [{b['start']:5d}-{b['end']:5d}] {b['ex']:9.0f} x {b['n']:4d}  inst {100 * b['ex'] * b['n'] / tex:5.1f}%"
              f"  stall {100 * b['ss'] / tss:5.1f}%  {b['first'][:50]}")


if __name__ == "__main__":
    main(*sys.argv[1:])
