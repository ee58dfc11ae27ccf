mkdir -p gpurun_out
: > gpurun_out/ctrlx.txt
for k in 1 2; do
for e in 0 1; do
for cfg in "--config layered-30 --precision double" "--config qft30"; do
  if [ $e = 1 ]; then export SVB_NO_CTRLX=1; else unset SVB_NO_CTRLX; fi
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "noctrlx=$e $cfg $r" >> gpurun_out/ctrlx.txt
done
done
done
unset SVB_NO_CTRLX
timeout 600 python bench.py --config layered33 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/bench_l33f.txt 2>&1
timeout 1500 python -m pytest tests/ -m gpu -x -q --timeout 900 > gpurun_out/pytest_ctrlx.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ctrlx.txt
