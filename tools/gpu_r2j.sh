mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multidevice.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for cfg in "4 8" "3 8" "4 4"; do set -- $cfg
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --streams $1 --gemm-warps $2 --pass-times > gpurun_out/bench_s$1_w$2.txt 2> gpurun_out/bench_s$1_w$2_passes.txt
done
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle and not prefix" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
