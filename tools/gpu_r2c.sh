mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle and not prefix" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --pass-times > gpurun_out/bench_gemm.txt 2> gpurun_out/bench_gemm_passes.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --streams 3 > gpurun_out/bench_gemm_s3.txt 2>&1
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --tensor-cores 2 > gpurun_out/bench_old.txt 2>&1
tail -2 gpurun_out/pytest_gpu.txt gpurun_out/pytest_scale.txt
