"""Summarize an ncu report: top stall reasons, DRAM bytes, pipe utilization and the hottest SASS lines.

python tools/ncu_stalls.py report.ncu-rep [n_top]
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
ntop = int(sys.argv[2]) if len(sys.argv) > 2 else 25
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(h, vals))
    print("==", d.get("Kernel Name", "")[:100])
    for k in ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
              "sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active",
              "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_bytes.sum",
              "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "launch__registers_per_thread"):
        if k in d:
            print(f"  {k} = {d[k]} {u[h.index(k)]}")
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v.replace(",", "") or 0)
          for k, v in d.items() if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")}
    tot = sum(st.values()) or 1
    print("  stalls:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:9]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
h = rows[1]
data = [r for r in rows[2:] if len(r) == len(h)]
ia, isrc, iss = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
tot = sum(float(r[iss] or 0) for r in data) or 1
for r in sorted(data, key=lambda r: -float(r[iss] or 0))[:ntop]:
    print(f"  {r[ia][-6:]} {float(r[iss] or 0) / tot * 100:5.1f}%  {r[isrc][:90]}")
