#!/bin/bash
# same-box A/B: c128 coefficient pool 80 KB (abtest/libsvb200_pool80.so) vs 64 KB (in-tree)
mkdir -p gpurun_out; : > gpurun_out/ab_pool.txt
for r in 1 2; do
  for L in paper_2604_03816_b200/lib/libsvb200.so abtest/libsvb200_pool80.so; do
    for a in "--config qft30" "--config layered-30 --precision double"; do
      echo "$L $a :: $(SVB_LIB=$L timeout 300 python bench.py --no-configs --no-cpu-baseline $a 2>/dev/null | tail -1 | cut -c1-260)" >> gpurun_out/ab_pool.txt
    done
  done
done
SVB_LIB=abtest/libsvb200_pool80.so timeout 900 python -m pytest tests/test_gpu_parity_scale.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "qft or QFT or c128 or double or w3 or width" > gpurun_out/pytest_pool80.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_pool80.txt
