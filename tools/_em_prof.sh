mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/em_launch.csv python bench.py --no-cpu --dense-steps 0 --steps 1 --warmup 1 --frames 200000 --em-utts 8192 > /dev/null 2>&1
