"""Summarise ncu reports (--page details + raw dram bytes) into profiles/.

    python scripts/ncu_summary.py <out.txt> <rep1.ncu-rep> [<rep2> ...]
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "L1/TEX Cache Throughput", "L2 Cache Throughput", "Compute (SM) Throughput", "Executed Ipc Active",
        "Issue Slots Busy", "Executed Instructions", "Warp Cycles Per Issued Instruction",
        "Avg. Active Threads Per Warp", "Registers Per Thread", "Achieved Occupancy", "Theoretical Occupancy",
        "Branch Efficiency", "Grid Size", "Block Size"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
       "sm__sass_inst_executed.sum", "smsp__sass_thread_inst_executed_op_fp32_pred_on.sum",
       "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct"]


def ncu_csv(rep, page):
    out = subprocess.run(["ncu", "-i", rep, "--page", page, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def summarise(rep):
    lines = []
    rows = ncu_csv(rep, "details")
    h = rows[0]
    ki, mi, vi, ui = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
    name = rows[1][ki] if len(rows) > 1 else "?"
    lines.append(f"kernel: {name}")
    seen = set()
    for r in rows[1:]:
        if r[mi] in KEYS and r[mi] not in seen:
            seen.add(r[mi])
            lines.append(f"  {r[mi]:40s} {r[vi]:>16s} {r[ui]}")
    raw = ncu_csv(rep, "raw")
    hdr, units, vals = raw[0], raw[1], raw[2]
    extra = {}
    for k in RAW:
        if k in hdr:
            i = hdr.index(k)
            lines.append(f"  {k:40s} {vals[i]:>16s} {units[i]}")
            extra[k] = (vals[i], units[i])
    return name, lines, extra


def to_bytes(v, u):
    v = float(v.replace(",", ""))
    return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)


if __name__ == "__main__":
    out = sys.argv[1]
    allines = []
    for rep in sys.argv[2:]:
        try:
            name, lines, extra = summarise(rep)
        except (ValueError, IndexError) as e:
            print(f"skip {rep}: {e}", file=sys.stderr)
            continue
        allines += [f"# {rep}"] + lines + [""]
        if "k_sweep" in name and "dram__bytes_read.sum" in extra:
            b = to_bytes(*extra["dram__bytes_read.sum"]) + to_bytes(*extra["dram__bytes_write.sum"])
            with open("profiles/sweep_traffic.json", "w") as f:
                json.dump({"kernel": name, "dram_bytes_per_launch": b, "source": rep}, f, indent=1)
    with open(out, "w") as f:
        f.write("\n".join(allines) + "\n")
    print("\n".join(allines))
