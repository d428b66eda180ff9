#!/bin/bash
# ncu launch list + full captures of the frame-posterior kernels on 1e6 frames (one GPU)
mkdir -p gpurun_out
B="python bench.py --no-cpu --no-em --dense-steps 0 --frames 1000000"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_align2.csv \
  $B --steps 2 --warmup 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_topk|grouped_ll|pair_scatter|pair_hist" -s 4 -c 4 \
  -o gpurun_out/prof_align2 $B --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out
