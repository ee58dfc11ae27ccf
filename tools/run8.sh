mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
for a in "--config layered-30 --precision double --streams 3" "--config qft30 --streams 3" "--config layered-30 --precision double"; do
  echo "ARGS $a :: $(timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "plan_shapes and double" > gpurun_out/pt_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pt_gpu.txt
