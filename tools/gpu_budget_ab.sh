#!/bin/bash
# c128 default cost budget A/B (5 vs 12): layered-33, layered-30, qft-30 and the Table-2 workload
mkdir -p gpurun_out
for b in 0 12; do
  for a in "--config layered-33 --precision double --steps 3" "--config layered-30 --precision double" "--config qft30"; do
    echo "B=$b $a :: $(timeout 600 python bench.py --no-configs --no-cpu-baseline --cost-budget $b $a 2>/dev/null | tail -1 | cut -c1-400)" >> gpurun_out/budget_ab.txt
  done
  PRECS=double PLAN_OPTS="cost_budget=$b.0" timeout 600 python tools/table2_probe.py 28 30 > gpurun_out/t2_budget_$b.txt 2>&1
done
