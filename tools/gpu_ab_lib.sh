#!/bin/bash
# same-box A/B of two builds of libsvb200 on config 2 (SVB_LIB selects the library)
mkdir -p gpurun_out; : > gpurun_out/ab_lib.txt
for r in 1 2 3; do
  for L in paper_2604_03816_b200/lib/libsvb200.so abtest/libsvb200_v5.so; do
    echo "$L :: $(SVB_LIB=$L timeout 300 python bench.py --no-configs --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | cut -c1-200)" >> gpurun_out/ab_lib.txt
  done
done
