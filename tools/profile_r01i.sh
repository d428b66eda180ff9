#!/bin/bash
# Round-1 profiling pass after the preselection split (main tcgen05 kernel + warp-per-frame post kernel).
mkdir -p gpurun_out
B="python bench.py --no-cpu --dense-steps 0 --em-utts 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_align_v5.csv \
  $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_tc_kernel" -s 1 -c 1 \
  -o gpurun_out/prof_select_tc_v5 -f $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_post" -s 1 -c 1 \
  -o gpurun_out/prof_post_v5 -f $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"whiten_ll" -s 1 -c 1 \
  -o gpurun_out/prof_whiten_v5 -f $B --steps 1 --warmup 1 --frames 1000000 > /dev/null 2>&1
python bench.py > gpurun_out/bench_r01i.json 2> gpurun_out/bench_r01i.err
ls -la gpurun_out/
