mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
rm -f gpurun_out/sweep.txt
for a in "" "--config layered-30" "--config qft-28 --precision single" "--config layered-26"; do
  echo "ARGS $a :: $(timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
