"""Summarize ncu captures (gpurun_out/*.ncu-rep) and launch lists into profiles/.

    python tools/summarize_ncu.py OUT_PREFIX rep1.ncu-rep[:frames] ... [--launches list.csv ...]

For each kernel in each report: duration, DRAM bytes, DMMA (FP64 tensor) utilisation, registers,
occupancy limits; `frames` (optional) normalizes DRAM bytes per frame for bench.py's `traffic`.
Launch lists (`ncu --metrics gpu__time_duration.sum --csv`) are aggregated into per-kernel shares.
"""

from __future__ import annotations

import collections
import csv
import io
import json
import subprocess
import sys

METRICS = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active": "dmma_pct_of_peak",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "launch__registers_per_thread": "registers",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts",
    "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_mem_active_pct",
    "l1tex__m_xbar2l1tex_read_bytes.sum": "l2_to_sm",
    "sm__inst_executed_pipe_tensor_subpipe_hmma.avg.pct_of_peak_sustained_active": "hmma_inst_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": "tensor_cycles_active_pct",
    "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active": "tc_cycles_active_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "smem_tc_wavefronts_pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed": "l2_throughput_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0,
         "second": 1e3, "ns": 1e-6, "us": 1e-3, "ms": 1.0, "s": 1e3}


def report(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for vals in rows[2:]:
        k = {"kernel": vals[hdr.index("Kernel Name")].split("(")[0].replace("void ", "")}
        for m, name in METRICS.items():
            if m not in hdr:
                continue
            i = hdr.index(m)
            try:
                v = float(vals[i].replace(",", ""))
            except ValueError:
                continue
            u = units[i]
            if name == "duration":
                v *= SCALE.get(u, 1.0)  # -> ms
                name = "duration_ms"
            elif (name.startswith("dram_") or name == "l2_to_sm") and not name.endswith("pct"):
                v *= SCALE.get(u, 1.0)  # -> bytes
                name += "_bytes"
            k[name] = v
        out.append(k)
    return out


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    hdr, data = rows[hi], rows[hi + 1:]
    kn, mv, mu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in data:
        if len(r) <= mv:
            continue
        v = float(r[mv].replace(",", "")) * SCALE.get(r[mu], 1.0)
        name = r[kn].split("(")[0].replace("void ", "")
        agg[name][0] += 1
        agg[name][1] += v
    tot = sum(v[1] for v in agg.values())
    return [{"kernel": k, "launches": v[0], "ms": v[1], "share": v[1] / tot}
            for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])]


def main():
    args = sys.argv[1:]
    prefix = args.pop(0)
    reps, lists = [], []
    while args:
        a = args.pop(0)
        if a == "--launches":
            lists.append(args.pop(0))
        else:
            reps.append(a)
    summary = {"reports": {}, "launch_lists": {}}
    for r in reps:
        path, _, frames = r.partition(":")
        ks = report(path)
        if frames:
            for k in ks:
                if "dram_read_bytes" in k:
                    k["dram_bytes_per_frame"] = (k["dram_read_bytes"] + k.get("dram_write_bytes", 0)) / float(frames)
        summary["reports"][path.split("/")[-1]] = ks
    for lpath in lists:
        summary["launch_lists"][lpath.split("/")[-1]] = launches(lpath)
    with open(prefix + ".json", "w") as fh:
        json.dump(summary, fh, indent=1)
    print(json.dumps(summary, indent=1)[:4000])


if __name__ == "__main__":
    main()
