# config-2 A/B over SVB_GEMM_DEBUG variants: bash tools/gpu_dbg.sh "0 4 2048 4096 ..."
mkdir -p gpurun_out
: > gpurun_out/dbg.txt
for k in 1 2; do
  for d in $1; do
    r=$(SVB_GEMM_DEBUG=$d timeout 300 python bench.py --no-cpu-baseline --no-configs --steps 10 --warmup 3 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
    echo "dbg=$d $r" >> gpurun_out/dbg.txt
  done
done
