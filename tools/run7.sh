mkdir -p gpurun_out
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --tensor-cores 1 --pass-times > gpurun_out/b_tc.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_tc_pass" -s 3 -c 1 \
  -o gpurun_out/prof_tc python bench.py --steps 1 --warmup 0 --no-cpu-baseline --tensor-cores 1 > gpurun_out/prof_tc.log 2>&1
