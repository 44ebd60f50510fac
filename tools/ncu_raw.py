"""Selected raw metrics of every kernel in an ncu report: python tools/ncu_raw.py rep [metric-substrings...]"""
import csv, subprocess, sys
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h, units = rows[0], rows[1]
keys = sys.argv[2:] or ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
                        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
                        "sm__inst_executed_pipe_fma", "smsp__inst_executed.sum", "launch__registers_per_thread",
                        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
                        "lts__t_bytes.sum"]
for r in rows[2:]:
    print(r[h.index("Kernel Name")][:90])
    for k in keys:
        for i, name in enumerate(h):
            if name == k or (k.endswith("*") and name.startswith(k[:-1])):
                print(f"   {name} = {r[i]} {units[i]}")
