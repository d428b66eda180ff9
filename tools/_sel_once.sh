mkdir -p gpurun_out
python tools/timeline_select.py > gpurun_out/tl.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:select_tc_kernel -c 1 -o gpurun_out/sel_full -f python tools/run_select_once.py > gpurun_out/ncu_sel.log 2>&1
