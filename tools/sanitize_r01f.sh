mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --leak-check no python tools/sanitize_small.py > gpurun_out/san_mem.txt 2>&1
timeout 900 $S --tool racecheck --racecheck-report all python tools/sanitize_small.py > gpurun_out/san_race.txt 2>&1
timeout 900 $S --tool synccheck python tools/sanitize_small.py > gpurun_out/san_sync.txt 2>&1
timeout 900 $S --tool memcheck --leak-check no python -c "
import sys; sys.path.insert(0,'.'); sys.path.insert(0,'tests/golden')
import numpy as np, cases, paper_1906_08556_b200 as pkg
x = cases.ubm_frames(cases.UBM_CASES[1])
d = pkg.train_gmm_diag(x, 16, n_iters=2, seed=3); f = pkg.train_gmm_full(x, d, n_iters=2); print('ubm ok')
" > gpurun_out/san_ubm.txt 2>&1
