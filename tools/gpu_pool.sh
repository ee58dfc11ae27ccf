#!/bin/bash
# c128 coefficient pool in global memory: QFT parity + config-3 timing
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qft or QFT or diag or c128 or double" > gpurun_out/pytest_pool.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pool.txt
timeout 600 python bench.py --config qft30 --no-configs --no-cpu-baseline --pass-times > gpurun_out/bench_qft_pool.txt 2>&1
timeout 600 python bench.py --config layered-30 --precision double --no-configs --no-cpu-baseline > gpurun_out/bench_l30_pool.txt 2>&1
