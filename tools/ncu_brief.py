"""Key metrics of every kernel in an ncu report: duration, pipes, occupancy, stalls.

    python tools/ncu_brief.py gpurun_out/pk/prof.ncu-rep
"""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "dur",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma%",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active": "fp64%",
    "sm__warps_active.avg.per_cycle_active": "warps/SM",
    "launch__registers_per_thread": "regs",
    "sm__inst_issued.avg.pct_of_peak_sustained_active": "issue%",
    "dram__bytes_read.sum": "dram_rd",
    "dram__bytes_write.sum": "dram_wr",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_conf",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": "smem_wf",
}
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h, u = rows[0], rows[1]
for r in rows[2:]:
    d = dict(zip(h, r))
    print("==", d.get("Kernel Name", "")[:80])
    print("  ", ", ".join(f"{v}={d.get(k, '?')}" for k, v in KEYS.items()))
    st = sorted(((float(d[k].replace(",", "")), k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")])
                 for k in h if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")
                 and d.get(k, "") not in ("", "n/a")), reverse=True)[:7]
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in st))
