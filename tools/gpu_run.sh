#!/bin/bash
# generic GPU-box runner: ensure the library is built for this snapshot, then run "$@"
mkdir -p gpurun_out
python -m paper_1906_08556_b200.build > gpurun_out/build.txt 2>&1 || { cat gpurun_out/build.txt; exit 1; }
"$@"
