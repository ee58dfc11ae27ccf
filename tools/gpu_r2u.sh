mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not qft30 and not 32q" > gpurun_out/pytest_u.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_u.txt
for d in 0 512 0 512; do
  SVB_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_u_$d.txt 2>&1
  grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_u_$d.txt | head -1 >> gpurun_out/bench_u_summary.txt
done
