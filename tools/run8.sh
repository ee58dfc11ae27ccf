mkdir -p gpurun_out
rm -f gpurun_out/sweep.txt
for a in "" "--config qft30" "--config layered-30 --precision double" "--tensor-cores -1"; do
  echo "ARGS $a :: $(timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
timeout 500 python tools/probe_phase.py SINGLE > gpurun_out/probe_phase_mma.txt 2>&1
