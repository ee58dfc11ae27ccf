#!/bin/bash
# bench parameter sweep (no cpu baseline); each line prefixed by its args
mkdir -p gpurun_out
OUT=gpurun_out/sweep.txt; : > $OUT
while read -r args; do
  [ "$args" = "-" ] && args=""
  line=$(timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $args 2>&1 | tail -1)
  echo "ARGS $args :: $line" >> $OUT
done < ${1:-tools/sweep_args.txt}
