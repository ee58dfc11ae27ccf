#!/bin/bash
# same-box A/B of library builds on config 2 and qft-30 (SVB_LIB selects the library)
mkdir -p gpurun_out; : > gpurun_out/ab_lib3.txt
for r in 1 2 3; do
  for L in paper_2604_03816_b200/lib/libsvb200.so abtest/libsvb200_al64.so; do
    echo "$L :: $(SVB_LIB=$L timeout 300 python bench.py --no-configs --no-cpu-baseline --steps 20 2>/dev/null | tail -1 | cut -c1-200)" >> gpurun_out/ab_lib3.txt
  done
done
for L in paper_2604_03816_b200/lib/libsvb200.so abtest/libsvb200_al64.so; do
  echo "$L qft30 :: $(SVB_LIB=$L timeout 300 python bench.py --config qft30 --no-configs --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200)" >> gpurun_out/ab_lib3.txt
  echo "$L layered-30 :: $(SVB_LIB=$L timeout 300 python bench.py --config layered-30 --precision double --no-configs --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-200)" >> gpurun_out/ab_lib3.txt
done
