# Round-2 ncu captures (run under gpurun from the repo root): one --set full capture per hot kernel and
# the launch list of the default bench command.  Summaries: python tools/summarize_ncu.py / ncu_stalls.py.
set -x
mkdir -p gpurun_out
N="ncu --set full --clock-control none --import-source on"
timeout 600 $N -k regex:"whiten_ll_kernel" -c 1 -o gpurun_out/r02_whiten python tools/align_once.py 2000000 > /dev/null 2>&1
timeout 600 $N -k regex:"select_tc_kernel|select_post_kernel" -c 2 -o gpurun_out/r02_select python tools/select_once.py 2000000 1 > /dev/null 2>&1
timeout 600 $N -k regex:"gemm_i8_kernel|split_tile_kernel" -c 3 -o gpurun_out/r02_i8 python tools/ozaki_once.py A > /dev/null 2>&1
timeout 600 $N -k regex:"sweep_posterior_kernel" -c 1 -o gpurun_out/r02_sweep python tools/post_bench.py 2048 400 > /dev/null 2>&1
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches_bench.csv \
  python bench.py --steps 2 --warmup 1 > gpurun_out/r02_launches_bench.log 2>&1
ls -la gpurun_out
