mkdir -p gpurun_out
( cd tools/probes && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu && ./dmma_probe ) > gpurun_out/dmma_probe.txt 2>&1
timeout 1500 python -m pytest tests/test_gpu_parity_scale.py -m gpu -q --timeout 900 -rs --durations=15 > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
