mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_align.py -x -q > gpurun_out/gpu_tests.log 2>&1
timeout 300 python tools/time_select_tc.py > gpurun_out/sel_dbg.log 2>&1
timeout 300 python tools/timeline_select.py 6 7 >> gpurun_out/sel_dbg.log 2>&1
