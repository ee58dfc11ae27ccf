mkdir -p gpurun_out
for a in "--config layered-30 --precision double" "--config qft30" ""; do
  echo "ARGS $a :: $(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
