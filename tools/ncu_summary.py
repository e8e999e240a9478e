"""Summarise an .ncu-rep (details page) into a compact text table (run here, no GPU)."""
import csv
import subprocess
import sys

KEYS = ("Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Executed Ipc Active", "Issue Slots Busy", "Warp Cycles Per Issued Instruction",
        "Eligible Warps Per Scheduler", "Executed Instructions", "Block Limit Registers", "Block Limit Shared Mem",
        "Dynamic Shared Memory Per Block", "Grid Size", "Block Size", "FP64 Pipe Utilization", "Mem Busy")


def main(path, out=None):
    txt = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    hdr = rows[0]
    lines = []
    seen = set()
    for r in rows[1:]:
        if len(r) < 15:
            continue
        name = r[4][:70]
        if name not in seen:
            lines.append(f"== {name}")
            seen.add(name)
        if r[12] in KEYS:
            lines.append(f"  {r[12]:42s} {r[14]:>14s} {r[13]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    if rr:
        h = rr[0]
        want = [i for i, k in enumerate(h) if k in ("dram__bytes_read.sum", "dram__bytes_write.sum",
                                                       "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                                                       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                                                       "smsp__inst_executed.sum", "gpu__time_duration.sum")]
        kn = h.index("Kernel Name") if "Kernel Name" in h else None
        for r in rr[2:]:
            label = f"[{r[kn].split('(')[0].split('::')[-1][:60]}] " if kn is not None else ""
            lines.append(f"  raw: {label}" + ", ".join(f"{h[i]}={r[i]}{rr[1][i]}" for i in want))
    text = "\n".join(lines)
    if out:
        open(out, "w").write(f"# ncu --set full summary of {path}\n" + text + "\n")
    print(text)


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else None)
