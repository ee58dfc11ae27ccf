mkdir -p gpurun_out
: > gpurun_out/bench_x_summary.txt
for d in 0 8192 0 8192; do
  SVB_GEMM_DEBUG=$d timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_x_$d.txt 2>&1
  echo "$d $(grep -o '"ms_per_step": [0-9.]*' gpurun_out/bench_x_$d.txt | head -1)" >> gpurun_out/bench_x_summary.txt
done
PRECS=double,single timeout 300 python tools/table2_probe.py 28 30 > gpurun_out/t2_x.txt 2>&1
timeout 1200 python -m pytest tests/ -m gpu -x -q --timeout 900 > gpurun_out/pytest_x.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_x.txt
