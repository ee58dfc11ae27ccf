# A/B over several library variants: bash tools/gpu_abn.sh "v1 v2 ..." <bench args>
mkdir -p gpurun_out
VS=$1; shift
for k in 1 2; do
  for lib in default $VS; do
    if [ $lib = default ]; then L=""; else L=$PWD/tmp_variants/$lib/libsvb200.so; fi
    r=$(SVB_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-configs "$@" 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
    echo "$lib $* $r" >> gpurun_out/abn.txt
  done
done
