mkdir -p gpurun_out
: > gpurun_out/sp_ab.txt
for k in 1 2; do
  for e in 0 1; do
    for cfg in "--config layered-30 --precision double" "--config qft30"; do
      if [ $e = 1 ]; then export SVB_NO_SPARSE2=1; else unset SVB_NO_SPARSE2; fi
      r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
      echo "nosparse=$e $cfg $r" >> gpurun_out/sp_ab.txt
    done
  done
done
unset SVB_NO_SPARSE2
timeout 300 python tools/pass_probe.py layered30 > gpurun_out/pp_sp.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 900 -k "not 32q" > gpurun_out/pytest_sp.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_sp.txt
