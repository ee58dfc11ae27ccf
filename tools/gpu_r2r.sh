mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multidevice.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --config layered-30 --precision double --steps 5 --warmup 2 --no-cpu-baseline --no-configs --pass-times > gpurun_out/bench_c128_f.txt 2> gpurun_out/bench_c128_f_passes.txt
timeout 300 python bench.py --config qft30 --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_qft_f.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
