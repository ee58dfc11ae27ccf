mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 -k "sharded or qft18" > gpurun_out/pt_new.txt 2>&1; echo "rc=$?" >> gpurun_out/pt_new.txt
