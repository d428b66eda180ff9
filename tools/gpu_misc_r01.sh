#!/bin/bash
# smoke(), reference arm, torchrun N=1 path, EM-kernel ncu captures
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ref.json 2> gpurun_out/ref.err; tail -1 gpurun_out/ref.json | cut -c1-400
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29511 \
  bench.py --gpus 1 --steps 2 --warmup 3 --frames 2000000 --em-utts 2048 --em-steps 1 --dense-steps 0 --no-cpu \
  > gpurun_out/torchrun1.json 2> gpurun_out/torchrun1.err; tail -1 gpurun_out/torchrun1.json | cut -c1-300
B="python bench.py --no-cpu --dense-steps 0 --frames 100000 --steps 1 --warmup 1 --em-utts 2048 --em-steps 1 --em-warmup 0"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_em2.csv $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"posterior_kernel|spd_solve_rows|bw_first|bw_second|sigma_floor" -c 5 \
  -o gpurun_out/prof_em2 $B > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gemm_kernel" -s 30 -c 4 \
  -o gpurun_out/prof_gemm2 $B > /dev/null 2>&1
ls -la gpurun_out | tail -12
