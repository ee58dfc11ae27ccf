"""Where the time of the paper's Table-2 workload goes on the device:
wall time of B200Engine.run_circuit vs device time of the plan and of each
pass.  usage: python tools/table2_probe.py [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_03816_b200 import B200Engine, Precision  # noqa: E402
from paper_2604_03816_b200 import generators as gen  # noqa: E402

eng = B200Engine("probe")
for n in [int(x) for x in sys.argv[1:]] or [28]:
    c = gen.random_su2_circuit(n, 10 * n, n)
    for prec in (Precision.DOUBLE, Precision.SINGLE):
        plan = eng.plan(c, prec)
        st = eng.init_state(n, prec)
        s = eng.stream()
        for _ in range(2):
            plan.execute(st.tensor, s)
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(plan.num_passes + 1)]
        cs = torch.cuda.ExternalStream(s)
        with torch.cuda.stream(cs):
            ev[0].record(cs)
            for p in range(plan.num_passes):
                plan.execute(st.tensor, s, p, 1)
                ev[p + 1].record(cs)
        torch.cuda.synchronize()
        per = [ev[p].elapsed_time(ev[p + 1]) for p in range(plan.num_passes)]
        eng.release(st)
        walls = []
        for _ in range(5):
            t0 = time.perf_counter()
            x = eng.run_circuit(c, prec)
            walls.append(time.perf_counter() - t0)
            eng.release(x)
        walls.sort()
        info = [plan.native.pass_info(p) for p in range(plan.num_passes)]
        print(f"n={n} {prec.value}: passes {plan.num_passes} device {sum(per):.2f} ms, run_circuit wall median "
              f"{1e3 * walls[2]:.2f} ms; per pass ms " +
              " ".join(f"{t:.2f}({i['num_gates']}g,{i['kernel']},{i['num_phases']}ph)" for t, i in zip(per, info)))
