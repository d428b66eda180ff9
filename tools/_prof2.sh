mkdir -p gpurun_out
B="python bench.py --no-cpu --dense-steps 0 --em-utts 0"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"whiten_ll" -s 8 -c 1 \
  -o gpurun_out/prof_whiten -f $B --steps 1 --warmup 1 --frames 1000000 > gpurun_out/p1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"select_post" -s 2 -c 1 \
  -o gpurun_out/prof_post -f $B --steps 1 --warmup 1 --frames 1000000 > gpurun_out/p2.log 2>&1
