#!/bin/bash
# first GPU contact: FP64 pipe ceilings, cuBLAS DGEMM peak, alignment parity tests
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/smi.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp64_peak tools/fp64_peak.cu && timeout 120 /tmp/fp64_peak > gpurun_out/fp64_peak.txt 2>&1
timeout 300 python tools/probe_box.py > gpurun_out/probe.json 2>&1
timeout 600 python -m pytest tests/test_gpu_align.py -q -x > gpurun_out/pytest_align.txt 2>&1
cat gpurun_out/smi.txt gpurun_out/fp64_peak.txt gpurun_out/probe.json; tail -30 gpurun_out/pytest_align.txt
