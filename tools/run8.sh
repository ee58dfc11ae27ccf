mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "plan_shapes" > gpurun_out/pt_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pt_gpu.txt
rm -f gpurun_out/sweep.txt
for a in "" "--streams 3" "--streams 3 --stages 6" "--config layered-30 --streams 3"; do
  echo "ARGS $a :: $(timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
