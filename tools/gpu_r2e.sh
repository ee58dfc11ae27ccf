mkdir -p gpurun_out
for s in 4 3 2; do
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --streams $s --pass-times > gpurun_out/bench_gemm_s$s.txt 2> gpurun_out/bench_gemm_s${s}_passes.txt
done
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_pass" -s 1 -c 3 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --streams 3 > gpurun_out/prof_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep "gemm passes 1-3 layered-28 streams 3" > gpurun_out/prof_gemm.txt 2>&1
