mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for d in 0 2048; do
SVB_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --pass-times > gpurun_out/bench_dbg$d.txt 2> gpurun_out/bench_dbg${d}_passes.txt
done
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle and not prefix" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
