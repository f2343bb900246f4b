"""Key metrics per kernel from an `ncu --page raw --csv` export: python tools/ncu_keys.py raw.csv [kernel regex]"""
import csv
import re
import sys

rows = list(csv.reader(open(sys.argv[1])))
pat = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
h, units = rows[0], rows[1]
KEYS = ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__occupancy_limit_registers",
        "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__inst_issued.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
        "smsp__thread_inst_executed_per_inst_executed.ratio"]
stall = [k for k in h if k.startswith("smsp__average_warp") and "issue_stalled" in k and k.endswith(".ratio")
         and "not_issued" not in k]
for r in rows[2:]:
    name = r[h.index("Kernel Name")]
    if pat and not pat.search(name):
        continue
    print("==", name[:70])
    for k in KEYS:
        if k in h and r[h.index(k)] not in ("", "n/a"):
            print(f"   {k:72s} {r[h.index(k)]:>16s} {units[h.index(k)]}")
    st = sorted(((float(r[h.index(k)] or 0), k) for k in stall), reverse=True)[:6]
    print("   stall cycles per issue:", ", ".join(f"{k.split('issue_stalled_')[1].replace('_per_issue_active.ratio', '')}={v:.2f}" for v, k in st))
