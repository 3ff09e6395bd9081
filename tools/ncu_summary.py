"""Summarise an ncu report: per kernel time, DRAM bytes, throughput, pipes, stalls."""
import csv, subprocess, sys, io
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[0]
want = {
    "name": "Kernel Name", "ms": "gpu__time_duration.sum", "rd": "dram__bytes_read.sum", "wr": "dram__bytes_write.sum",
    "dram%": "dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm%": "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "issue%": "sm__inst_issued.avg.pct_of_peak_sustained_active", "fma%": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "warps%": "sm__warps_active.avg.pct_of_peak_sustained_active", "regs": "launch__registers_per_thread",
    "occ_reg": "launch__occupancy_limit_registers", "occ_smem": "launch__occupancy_limit_shared_mem",
    "bank_conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "inst": "smsp__inst_executed.sum",
    "local_ld": "l1tex__t_sectors_pipe_lsu_mem_local_op_ld.sum",
}
idx = {k: (hdr.index(v) if v in hdr else None) for k, v in want.items()}
units = rows[1]
for r in rows[2:]:
    d = {k: (r[i] if i is not None else "-") for k, i in idx.items()}
    print(" | ".join(f"{k}={d[k]}" for k in want))
