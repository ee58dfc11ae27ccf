mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q --timeout 300 > gpurun_out/pytest_gpu.txt 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.txt
timeout 300 python bench.py --config qft30 --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_qft.txt 2>&1
timeout 300 python bench.py --config layered-30 --precision double --steps 5 --warmup 2 --no-cpu-baseline --no-configs > gpurun_out/bench_l30.txt 2>&1
# paper Table 2 workload (random SU(2), 10n gates) through this package's CLI
timeout 600 python -m paper_2604_03816_b200 bench-scaling --qubits 14,16,18,20,22,24,26,28,30 --repetitions 5 > gpurun_out/table2_b200.json 2> gpurun_out/table2_b200.err
# and through the reference's own CLI with "b200" registered (fidelity vs aqsim's reference engine)
timeout 900 python -c "
import sys; sys.path.append('baseline/_ref')
import paper_2604_03816_b200
from aqsim.cli import main
sys.exit(main(['bench-scaling', '--qubits', '14,16,18,20,22', '--engines', 'b200,parallel', '--repetitions', '3', '--format', 'json']))
" > gpurun_out/table2_aqsim_cli.json 2> gpurun_out/table2_aqsim_cli.err
