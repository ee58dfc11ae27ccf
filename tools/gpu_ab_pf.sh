#!/bin/bash
# same-box A/B: c128 op-dispatch prefetch (abtest/libsvb200_pf.so) vs base
mkdir -p gpurun_out; : > gpurun_out/ab_pf.txt
for r in 1 2; do
  for L in abtest/libsvb200_base.so abtest/libsvb200_pf.so; do
    for a in "--config layered-30 --precision double" "--config qft30" "--config layered-33 --precision double --steps 3"; do
      echo "$L $a :: $(SVB_LIB=$L timeout 300 python bench.py --no-configs --no-cpu-baseline $a 2>/dev/null | tail -1 | cut -c1-200)" >> gpurun_out/ab_pf.txt
    done
  done
done
SVB_LIB=abtest/libsvb200_pf.so timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qft or QFT or c128 or double or layered" > gpurun_out/pytest_pf.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pf.txt
