mkdir -p gpurun_out
: > gpurun_out/ctrl.txt
for k in 1 2; do
for cfg in "--config layered-30 --precision double" "--config qft30"; do
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "$cfg $r" >> gpurun_out/ctrl.txt
done
done
timeout 600 python bench.py --config layered33 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/bench_l33d.txt 2>&1
timeout 1500 python -m pytest tests/ -m gpu -x -q --timeout 900 > gpurun_out/pytest_ctrl.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ctrl.txt
