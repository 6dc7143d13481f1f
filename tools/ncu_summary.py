"""Summary rows of an ncu --set full capture (dev tool).

usage: python tools/ncu_summary.py gpurun_out/prof_TAG.ncu-rep > profiles/rNN_ncu_full.csv

One row per captured launch: time, DRAM bytes, DRAM throughput, issue
activity, warps active, registers, shared-memory occupancy limit,
instructions and shared-memory wavefronts (`ncu -i ... --page raw --csv`)."""
import csv
import io
import subprocess
import sys

COLS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_shared_mem", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum"]

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units, data = rows[0], rows[1], rows[2:]
idx = [hdr.index(c) for c in COLS]
w = csv.writer(sys.stdout, lineterminator="\n")
w.writerow(COLS)
w.writerow([units[i] for i in idx])
for r in data:
    w.writerow([r[i] for i in idx])
