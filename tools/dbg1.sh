mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -v --timeout 100 -k "plan_shapes" -x > gpurun_out/pt_shapes.txt 2>&1; echo "rc=$?" >> gpurun_out/pt_shapes.txt
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --tensor-cores 1 --cost-budget 2.0 > gpurun_out/tc_b2.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_b2.txt
timeout 120 python bench.py --steps 2 --warmup 3 --no-cpu-baseline --tensor-cores 1 --tc-min-dense 3 > gpurun_out/tc_md3.txt 2>&1; echo "rc=$?" >> gpurun_out/tc_md3.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -v --timeout 300 --durations=0 -k "not plan_shapes" > gpurun_out/pt_rest.txt 2>&1; echo "rc=$?" >> gpurun_out/pt_rest.txt
