mkdir -p gpurun_out
: > gpurun_out/beam.txt
for k in 1 2; do
for cfg in "" "--config qft30" "--config layered-30 --precision double"; do
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "$cfg $r" >> gpurun_out/beam.txt
done
done
timeout 600 python bench.py --config layered33 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/bench_l33b.txt 2>&1
timeout 1500 python -m pytest tests/ -m gpu -x -q --timeout 900 > gpurun_out/pytest_beam.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_beam.txt
