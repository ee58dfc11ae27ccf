mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python __graft_entry__.py --smoke > gpurun_out/smoke.txt 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.txt
rm -f gpurun_out/sweep.txt
for a in "--config qft30" "--config layered33" "--config layered-30 --precision double" "--config layered-30" "--config qft-28 --precision single"; do
  echo "ARGS $a :: $(timeout 400 python bench.py --steps 5 --warmup 3 --no-cpu-baseline $a 2>&1 | tail -1)" >> gpurun_out/sweep.txt
done
timeout 600 python bench.py > gpurun_out/bench_default.txt 2>&1
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_(tile|reg|tc)_pass" -c 40 --csv --log-file gpurun_out/launches.csv python bench.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/ncu_launch.log 2>&1
bash tools/ncu_full.sh 3 prof_final
