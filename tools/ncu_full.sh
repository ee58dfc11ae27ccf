#!/bin/bash
# Full ncu capture of one tile-pass launch (arg1: skip count, arg2: output name, rest: bench args)
mkdir -p gpurun_out
SKIP=${1:-1}; NAME=${2:-prof}; shift 2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_(tile|reg|gemm)_pass" -s $SKIP -c 1 \
  -o gpurun_out/$NAME python bench.py --steps 1 --warmup 0 --no-cpu-baseline "$@" > gpurun_out/$NAME.log 2>&1
echo "ncu rc=$?" >> gpurun_out/$NAME.log
