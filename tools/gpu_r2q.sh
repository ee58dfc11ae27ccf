mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity_scale.py -m gpu -q --timeout 900 -k "renormalisation" -s > gpurun_out/pytest_norenorm.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_norenorm.txt
timeout 300 python tools/pass_probe.py qft30 > gpurun_out/pp_q2.txt 2>&1
SVB_REG_STAGES=2 timeout 300 python tools/pass_probe.py qft30 >> gpurun_out/pp_q2.txt 2>&1
timeout 300 python tools/pass_probe.py layered30 >> gpurun_out/pp_q2.txt 2>&1
