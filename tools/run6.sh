mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for a in "--config qft30" "--config qft30 --cost-budget 10"; do
  echo "ARGS $a :: $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
bash tools/ncu_full.sh 1 prof_qft30c --config qft30
