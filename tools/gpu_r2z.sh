mkdir -p gpurun_out
bash tools/gpu_ab.sh split --config layered-30 --precision double --steps 5 --warmup 2
timeout 300 python tools/pass_probe.py qft30 > gpurun_out/pp_qft.txt 2>&1
SVB_REG_STAGES=2 timeout 300 python tools/pass_probe.py qft30 >> gpurun_out/pp_qft.txt 2>&1
PLAN_OPTS="streams=4" timeout 300 python tools/pass_probe.py qft30 >> gpurun_out/pp_qft.txt 2>&1
timeout 300 python tools/pass_probe.py layered30 >> gpurun_out/pp_qft.txt 2>&1
