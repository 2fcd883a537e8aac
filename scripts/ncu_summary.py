"""Summarise ncu reports (--page details + raw dram bytes) into profiles/.

    python scripts/ncu_summary.py [--workload NAME] [--outdir DIR] <out.txt> <rep1.ncu-rep> [<rep2> ...]

With --workload, also writes the per-workload records bench.py reads:
profiles/traffic_NAME.json (dram bytes of one k_sweep launch, its roofline
`traffic`) and profiles/instr_NAME.json (warp instructions, dram bytes and ncu
duration per captured kernel launch).
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


def to_us(v, u):
    v = float(v.replace(",", ""))
    return v * {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}.get(u, 1.0)


def short(name):
    return name.split("(")[0].replace("void ", "").split("<")[0].replace("sb::", "")


if __name__ == "__main__":
    args = sys.argv[1:]
    wl = None
    outdir = "profiles"
    while args and args[0].startswith("--"):
        if args[0] == "--workload":
            wl, args = args[1], args[2:]
        elif args[0] == "--outdir":
            outdir, args = args[1], args[2:]
        else:
            break
    out = args[0]
    allines = []
    instr = {}
    for rep in args[1:]:
        try:
            name, lines, extra = summarise(rep)
        except (ValueError, IndexError) as e:
            print(f"skip {rep}: {e}", file=sys.stderr)
            continue
        allines += [f"# {rep}"] + lines + [""]
        ins = None
        for ln in lines:
            if ln.strip().startswith("Executed Instructions"):
                ins = float(ln.split()[2].replace(",", ""))
        if "dram__bytes_read.sum" in extra and ins is not None:
            b = to_bytes(*extra["dram__bytes_read.sum"]) + to_bytes(*extra["dram__bytes_write.sum"])
            instr[short(name)] = {"warp_instr": ins,
                                  "dram_bytes": b, "us_ncu": to_us(*extra["gpu__time_duration.sum"]),
                                  "source": rep}
            if wl and "k_sweep" in name:
                with open(f"{outdir}/traffic_{wl}.json", "w") as f:
                    json.dump({"kernel": name, "dram_bytes_per_launch": b, "source": rep}, f, indent=1)
    if wl and instr:
        with open(f"{outdir}/instr_{wl}.json", "w") as f:
            json.dump(instr, f, indent=1)
    with open(out, "w") as f:
        f.write("\n".join(allines) + "\n")
    print("\n".join(allines))
