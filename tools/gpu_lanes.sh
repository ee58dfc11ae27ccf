mkdir -p gpurun_out
: > gpurun_out/lanes.txt
for k in 1 2; do
for cfg in "--config layered-30 --precision double" "--config qft30"; do
  r=$(timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 5 --warmup 2 $cfg 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
  echo "$cfg $r" >> gpurun_out/lanes.txt
done
done
timeout 600 python bench.py --config layered33 --steps 2 --warmup 1 --no-cpu-baseline --no-configs > gpurun_out/bench_l33e.txt 2>&1
timeout 900 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,gpu__time_duration.sum -k regex:"k_reg_pass" -s 3 -c 1 python bench.py --config layered-30 --precision double --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/lanes_ncu.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 900 -k "not 32q" > gpurun_out/pytest_lanes.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_lanes.txt
