mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config qft30 --pass-times > gpurun_out/b_qft30.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --config qft30 --cost-budget 10 > gpurun_out/b_qft30_b10.txt 2>&1
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/b_l28.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config layered33 > gpurun_out/b_l33.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --config layered33 --cost-budget 10 > gpurun_out/b_l33_b10.txt 2>&1
