"""Condense an ncu report into a small JSON summary for profiles/ (per launch).

    python tools/ncu_summary.py gpurun_out/x.ncu-rep profiles/x_summary.json
"""
import csv
import io
import json
import subprocess
import sys

METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
           "smsp__inst_executed.sum", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
           "lts__t_bytes.sum", "sm__pipe_tensor_op_imma_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__throughput.avg.pct_of_peak_sustained_elapsed", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
           "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "l1tex__m_xbar2l1tex_read_bytes.sum",
           # busy cycles (not instruction counts): IMAD / IMAD.HI / IMAD.WIDE issue only to fmaheavy
           "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed",
           "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active"]
rep, out = sys.argv[1], sys.argv[2]
txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(METRICS)],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
hdr, units = rows[0], rows[1]
res = []
for r in rows[2:]:
    d = {"kernel": r[hdr.index("Kernel Name")][:80]}
    for m in METRICS:
        if m in hdr:
            i = hdr.index(m)
            try:
                d[m] = float(r[i].replace(",", ""))
            except ValueError:
                d[m] = r[i]
            d[m + "_unit"] = units[i]
    res.append(d)
json.dump({"report": rep, "launches": res}, open(out, "w"), indent=1)
print(out, len(res), "launches")
