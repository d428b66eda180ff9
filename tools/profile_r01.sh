#!/bin/bash
# Round-1 profiling pass (one GPU): launch lists + full ncu captures of the top kernels.
set -x
mkdir -p gpurun_out
NCU=ncu
B="python bench.py --no-cpu"
# frame-posterior path: launch list (cold-cache, serialised: compare shares)
timeout 600 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_align.csv \
  $B --steps 2 --warmup 1 --frames 1000000 --no-em > /dev/null 2>&1
# dominant kernel, full set
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:full_ll_kernel -s 2 -c 1 \
  -o gpurun_out/prof_full_ll $B --steps 1 --warmup 1 --frames 1000000 --no-em > /dev/null 2>&1
timeout 600 $NCU --set full --clock-control none --import-source on -k regex:select_topk -s 2 -c 1 \
  -o gpurun_out/prof_select $B --steps 1 --warmup 1 --frames 1000000 --no-em > /dev/null 2>&1
# EM iteration: launch list on a 2048-utterance corpus, then full captures of its top kernels
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_em.csv \
  $B --steps 1 --warmup 1 --frames 100000 --em-utts 2048 --em-steps 1 --em-warmup 0 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:posterior_kernel -c 1 \
  -o gpurun_out/prof_posterior $B --steps 1 --warmup 1 --frames 100000 --em-utts 1024 --em-steps 1 --em-warmup 0 > /dev/null 2>&1
timeout 900 $NCU --set full --clock-control none --import-source on -k regex:gemm_kernel --launch-skip 40 -c 6 \
  -o gpurun_out/prof_gemm $B --steps 1 --warmup 1 --frames 100000 --em-utts 1024 --em-steps 1 --em-warmup 0 > /dev/null 2>&1
ls -la gpurun_out/
