mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; free -g >> gpurun_out/gpu.txt
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 -rs > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
bash tools/ncu_full.sh 3 prof_c128_l30 --config layered-30 --precision double
python tools/ncu_summary.py gpurun_out/prof_c128_l30.ncu-rep "layered-30 c128 pass 3" > gpurun_out/prof_c128_l30.txt 2>&1
