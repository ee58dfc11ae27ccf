mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle and not prefix" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --pass-times > gpurun_out/bench_gemm.txt 2> gpurun_out/bench_gemm_passes.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_pass" -s 1 -c 3 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/prof_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep "gemm passes 1-3 layered-28" > gpurun_out/prof_gemm.txt 2>&1
