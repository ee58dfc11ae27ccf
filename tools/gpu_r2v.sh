mkdir -p gpurun_out
: > gpurun_out/t2_opts.txt
for o in "" "min_low_bits=4" "min_low_bits=5" "min_low_bits=6" "cost_budget=10" ; do
  PLAN_OPTS="$o" PRECS=double timeout 200 python tools/table2_probe.py 28 30 >> gpurun_out/t2_opts.txt 2>&1
done
for o in "" "min_low_bits=5" "min_low_bits=6" "min_low_bits=7"; do
  PLAN_OPTS="$o" PRECS=single timeout 200 python tools/table2_probe.py 28 30 >> gpurun_out/t2_opts.txt 2>&1
done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multidevice.py -m gpu -x -q --timeout 600 -k "sharded or multidevice or Multi or shard" > gpurun_out/pytest_p2p.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_p2p.txt
