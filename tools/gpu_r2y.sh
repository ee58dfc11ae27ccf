mkdir -p gpurun_out
PRECS=double,single timeout 300 python tools/table2_probe.py 24 28 30 > gpurun_out/t2_y.txt 2>&1
bash tools/gpu_r2t.sh
timeout 1500 python -m pytest tests/ -m gpu -x -q --timeout 900 > gpurun_out/pytest_y.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_y.txt
