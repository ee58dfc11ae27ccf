mkdir -p gpurun_out
: > gpurun_out/ctrl2.txt
for k in 1 2; do
for e in 0 1; do
for cfg in "--config layered-30 --precision double" "--config qft30"; do
  if [ $e = 1 ]; then export SVB_NO_CTRL=1; else unset SVB_NO_CTRL; fi
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "noctrl=$e $cfg $r" >> gpurun_out/ctrl2.txt
done
done
done
unset SVB_NO_CTRL
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 900 > gpurun_out/pytest_ctrl2.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_ctrl2.txt
