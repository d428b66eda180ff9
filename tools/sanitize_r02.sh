# compute-sanitizer memcheck / racecheck / synccheck on tools/sanitize_r02.py (round-2 kernels)
mkdir -p gpurun_out
S=/usr/local/cuda/bin/compute-sanitizer
timeout 900 $S --tool memcheck --leak-check no python tools/sanitize_r02.py > gpurun_out/r02_san_mem.txt 2>&1
timeout 900 $S --tool racecheck --racecheck-report all python tools/sanitize_r02.py > gpurun_out/r02_san_race.txt 2>&1
timeout 900 $S --tool synccheck python tools/sanitize_r02.py > gpurun_out/r02_san_sync.txt 2>&1
for f in gpurun_out/r02_san_*.txt; do tail -n 2 $f; done
