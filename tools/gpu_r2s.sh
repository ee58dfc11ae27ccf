mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
for st in 2 1; do
SVB_REG_STAGES=$st timeout 300 python bench.py --config qft30 --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_qft_st$st.txt 2>&1
SVB_REG_STAGES=$st timeout 300 python bench.py --config layered-30 --precision double --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_l30_st$st.txt 2>&1
done
SVB_REG_STAGES=2 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-configs > gpurun_out/bench_c64_st2.txt 2>&1
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -x -q --timeout 600 -k "not full_size_vs_oracle and not prefix" > gpurun_out/pytest_scale.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_scale.txt
