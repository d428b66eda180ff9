mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_align.py -x -q > gpurun_out/gpu_tests.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/sel_launch.csv python tools/run_select_once.py 2000000 > /dev/null 2>&1
