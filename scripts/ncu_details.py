"""Key metrics of an ncu --set full report (.ncu-rep) per kernel, as text for profiles/."""
import csv
import subprocess
import sys

KEYS = ["Duration", "SM Frequency", "Elapsed Cycles", "Memory Throughput", "DRAM Throughput",
        "Compute (SM) Throughput", "L2 Hit Rate", "Registers Per Thread", "Achieved Occupancy", "Block Size",
        "Grid Size", "Dynamic Shared Memory Per Block", "Issue Slots Busy", "Executed Ipc Active",
        "Theoretical Occupancy", "Waves Per SM"]
RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
       "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "smsp__warps_active.avg.pct_of_peak_sustained_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "lts__t_bytes.sum"]


def main(path):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(det.splitlines()))
    hdr = rows[0]
    ki, mi, vi, ui, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
    seen = {}
    for r in rows[1:]:
        if r[mi] in KEYS:
            seen.setdefault((r[ii], r[ki][:70]), []).append(f"{r[mi]} = {r[vi]} {r[ui]}")
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    h, units = rr[0], rr[1]
    for n, ((kid, name), items) in enumerate(seen.items()):
        print(f"== [{kid}] {name}")
        for it in items:
            print("   ", it)
        if 2 + n < len(rr):
            vals = rr[2 + n]
            for key in RAW:
                if key in h:
                    print(f"    {key} = {vals[h.index(key)]} {units[h.index(key)]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print(f"# {p}")
        main(p)
