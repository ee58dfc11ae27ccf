# A/B of library variants: bash tools/gpu_ab.sh <variant dir under tmp_variants> <bench args...>
mkdir -p gpurun_out
V=$1; shift
echo "== $V $*" >> gpurun_out/ab_$V.txt
for k in 1 2; do
  for lib in default $V; do
    if [ $lib = default ]; then L=""; else L=$PWD/tmp_variants/$lib/libsvb200.so; fi
    r=$(SVB_LIB=$L timeout 300 python bench.py --no-cpu-baseline --no-configs "$@" 2>/dev/null | tail -1 | grep -o '"ms_per_step": [0-9.]*')
    echo "$lib $* $r" >> gpurun_out/ab_$V.txt
  done
done
