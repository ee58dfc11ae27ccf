mkdir -p gpurun_out
for d in 0 64 128; do
SVB_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --pass-times > gpurun_out/bench_dbg$d.txt 2> gpurun_out/bench_dbg${d}_passes.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_pass" -s 3 -c 1 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/prof_gemm.log 2>&1
ncu -i gpurun_out/prof_gemm.ncu-rep --page raw --csv > gpurun_out/prof_gemm_raw.csv 2>&1
