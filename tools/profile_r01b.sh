#!/bin/bash
# Round-1 profiling pass after the tcgen05 preselection + whitening kernels (one GPU).
mkdir -p gpurun_out
B="python bench.py --no-cpu --dense-steps 0 --em-utts 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_align_v2.csv \
  $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_tc_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_select_tc $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"whiten_ll" -s 8 -c 1 \
  -o gpurun_out/prof_whiten $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
ls -la gpurun_out/
