#!/bin/bash
# Round-2 evidence run: default bench line (config 2 + configs 3/4 + CPU
# baseline), the reference arm, the ncu launch list of one config-2 step and
# full captures of the dominant kernels (c64 gemm pass, c128 register pass).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_noise.py -m gpu -q > gpurun_out/pytest_noise.txt 2>&1; echo "rc=$?" >> gpurun_out/pytest_noise.txt
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/bench_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(tile|reg|gemm)_pass" -c 40 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gemm_pass" -s 3 -c 1 \
  -o gpurun_out/prof_gemm python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/prof_gemm.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_gemm.ncu-rep "k_gemm_pass<4> layered-28 c64 pass 3 (3 GEMMs), round 2 (final, r02_v6)" > gpurun_out/prof_gemm.txt 2>&1
python tools/ncu_opstall.py gpurun_out/prof_gemm.ncu-rep 0 16 >> gpurun_out/prof_gemm.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_reg_pass" -s 3 -c 1 \
  -o gpurun_out/prof_c128 python bench.py --config layered-30 --precision double --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/prof_c128.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_c128.ncu-rep "k_reg_pass<double2,4,7,3> layered-30 c128 pass 3, round 2 (r02_v6)" > gpurun_out/prof_c128.txt 2>&1
python tools/ncu_opstall.py gpurun_out/prof_c128.ncu-rep 0 16 >> gpurun_out/prof_c128.txt 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_reg_pass" -s 3 -c 1 \
  -o gpurun_out/prof_qft python bench.py --config qft30 --steps 1 --warmup 0 --no-cpu-baseline --no-configs > gpurun_out/prof_qft.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_qft.ncu-rep "k_reg_pass<double2,4,7,3> qft-30 c128 pass 3, round 2 (r02_v6)" > gpurun_out/prof_qft.txt 2>&1
python tools/ncu_opstall.py gpurun_out/prof_qft.ncu-rep 0 16 >> gpurun_out/prof_qft.txt 2>&1
tail -n 2 gpurun_out/bench_default.txt | cut -c1-300
