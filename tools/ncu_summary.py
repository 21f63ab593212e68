"""Summarise an ncu report: per-kernel duration, DRAM bytes and throughput."""
import csv, io, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = ["Kernel Name", "Grid Size", "Block Size", "gpu__time_duration.sum", "dram__bytes_read.sum",
        "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
        "launch__shared_mem_per_block_dynamic", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
units = rows[1]
for r in rows[2:]:
    d = {w: (r[hdr.index(w)], units[hdr.index(w)]) for w in want if w in hdr}
    name = d["Kernel Name"][0].split("(")[0]
    t = float(d["gpu__time_duration.sum"][0]); tu = d["gpu__time_duration.sum"][1]
    rd = float(d["dram__bytes_read.sum"][0]); ru = d["dram__bytes_read.sum"][1]
    wr = float(d["dram__bytes_write.sum"][0])
    print(f"{name:32s} grid={d['Grid Size'][0]:>12s} t={t:.2f}{tu} read={rd:.2f}{ru} write={wr:.2f} "
          f"dram%={d['gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed'][0]} "
          f"regs={d['launch__registers_per_thread'][0]} smem={d['launch__shared_mem_per_block_dynamic'][0]}{d['launch__shared_mem_per_block_dynamic'][1]} "
          f"warps%={d['sm__warps_active.avg.pct_of_peak_sustained_active'][0]}")
