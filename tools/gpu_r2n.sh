mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multidevice.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs --pass-times > gpurun_out/bench_gemm.txt 2> gpurun_out/bench_gemm_passes.txt
rm -f gpurun_out/gemm_trace.txt; SVB_GEMM_TRACE=1 timeout 200 python tools/gemm_trace.py 3 >> gpurun_out/gemm_trace.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
