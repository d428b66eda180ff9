#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"select_topk" -s 1 -c 1 \
  -o gpurun_out/prof_select3 python bench.py --no-cpu --no-em --dense-steps 0 --frames 1000000 --steps 1 --warmup 1 > /dev/null 2>&1
ls -la gpurun_out/prof_select3.ncu-rep
