mkdir -p gpurun_out
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_w.txt 2>&1
PRECS=double,single timeout 300 python tools/table2_probe.py 28 30 > gpurun_out/t2_w.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not 32q" > gpurun_out/pytest_w.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_w.txt
