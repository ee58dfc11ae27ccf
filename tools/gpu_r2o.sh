mkdir -p gpurun_out
for s in 3 4; do
timeout 300 python bench.py --config layered-30 --precision double --steps 5 --warmup 2 --no-cpu-baseline --no-configs --streams $s --pass-times > gpurun_out/bench_c128_s$s.txt 2> gpurun_out/bench_c128_s${s}_passes.txt
done
timeout 300 python bench.py --config qft30 --steps 5 --warmup 2 --no-cpu-baseline --no-configs --streams 4 > gpurun_out/bench_qft_s4.txt 2>&1
timeout 300 python bench.py --config qft30 --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_qft_s3.txt 2>&1
