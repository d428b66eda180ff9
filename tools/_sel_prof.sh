mkdir -p gpurun_out
for p in 65536,8,8,64,0 32768,8,4,64,0 65536,16,8,64,0; do echo "pipe $p" >> gpurun_out/sel_dbg.log; TVK_SEL_PIPE=$p timeout 300 python tools/time_select_tc.py >> gpurun_out/sel_dbg.log 2>&1; TVK_SEL_PIPE=$p timeout 300 python tools/timeline_select.py 6 >> gpurun_out/sel_dbg.log 2>&1; done
