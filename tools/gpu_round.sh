#!/bin/bash
# Full GPU suite + the evidence run (bench line, reference arm, ncu launch list and full captures)
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_gpu.txt
bash tools/gpu_evidence.sh
