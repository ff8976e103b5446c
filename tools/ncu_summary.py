"""Summarise an ncu report: key SOL / memory / occupancy metrics per kernel."""
import csv
import io
import subprocess
import sys

KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "L1/TEX Hit Rate",
        "Compute (SM) Throughput", "Executed Ipc Active", "Registers Per Thread",
        "Dynamic Shared Memory Per Block", "Block Limit Registers", "Block Limit Shared Mem",
        "Theoretical Occupancy", "Achieved Occupancy", "Eligible Warps Per Scheduler",
        "Issued Warp Per Scheduler", "Warp Cycles Per Issued Instruction"]
RAW = ["dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_bytes.sum",
       "gpu__time_duration.sum", "smsp__inst_executed.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[0]
    ki, mi, ui, vi = (hdr.index("Kernel Name"), hdr.index("Metric Name"),
                      hdr.index("Metric Unit"), hdr.index("Metric Value"))
    seen = {}
    for r in rows[1:]:
        if len(r) > vi and r[mi] in KEYS:
            seen.setdefault(r[ki][:60], {})[r[mi]] = f"{r[vi]} {r[ui]}"
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    for k, d in seen.items():
        print("kernel:", k)
        for key in KEYS:
            if key in d:
                print(f"  {key}: {d[key]}")
    if len(rr) > 2:
        h, u = rr[0], rr[1]
        for row in rr[2:]:
            for m in RAW:
                if m in h:
                    print(f"  {m}: {row[h.index(m)]} {u[h.index(m)]}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        main(p)
