mkdir -p gpurun_out
bash tools/sweep.sh
cat gpurun_out/sweep.txt | cut -c1-400
bash tools/ncu_full.sh 3 prof_l28c64 --cost-budget 5.0
bash tools/ncu_full.sh 3 prof_l30c128 --config layered-30 --precision double
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pass-times --cost-budget 5.0 > gpurun_out/pt_l28.txt 2>&1
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --pass-times --config layered-30 --precision double > gpurun_out/pt_l30d.txt 2>&1
