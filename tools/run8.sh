mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 120 > gpurun_out/pt_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pt_gpu.txt
timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --tensor-cores 2 --pass-times > gpurun_out/pt_mma.txt 2>&1
timeout 200 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --tensor-cores 2 --cost-budget 14 > gpurun_out/pt_mma14.txt 2>&1
