mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_pass" -s 1 -c 3 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/prof_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep "gemm passes 1-3 layered-28" > gpurun_out/prof_gemm.txt 2>&1
python tools/ncu_opstall.py gpurun_out/prof_gemm.ncu-rep > gpurun_out/prof_gemm_ops.txt 2>&1
