"""Where the time of the paper's Table-2 workload goes: wall time of each
step of B200Engine.run_circuit (plan lookup, allocation + |0>, execution,
synchronise) and the device time of each pass.
usage: python tools/table2_probe.py [n ...]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_03816_b200 import B200Engine, Precision  # noqa: E402
from paper_2604_03816_b200 import generators as gen  # noqa: E402


def wall(f):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = f()
    torch.cuda.synchronize()
    return r, 1e3 * (time.perf_counter() - t0)


# planner options from the environment, e.g. PLAN_OPTS="min_low_bits=5,cost_budget=8"
opts = {k: float(v) if "." in v else int(v) for k, v in
        (kv.split("=") for kv in os.environ.get("PLAN_OPTS", "").split(",") if kv)}
from paper_2604_03816_b200.b200 import plan_options  # noqa: E402
eng = B200Engine("probe", options=plan_options(**opts) if opts else None)
precs = [Precision(p) for p in os.environ.get("PRECS", "double,single").split(",")]
for n in [int(x) for x in sys.argv[1:]] or [28]:
    c = gen.random_su2_circuit(n, 10 * n, n)
    for prec in precs:
        plan, t_plan0 = wall(lambda: eng.plan(c, prec))
        plan, t_plan1 = wall(lambda: eng.plan(c, prec))
        st, t_init = wall(lambda: eng.init_state(n, prec))
        _, t_exec = wall(lambda: eng.execute(st, plan))
        _, t_exec2 = wall(lambda: eng.execute(st, plan))
        per = []
        for p in range(plan.num_passes):
            _, t = wall(lambda: plan.execute(st.tensor, eng.stream(), p, 1))
            per.append(t)
        _, t_rel = wall(lambda: eng.release(st))
        walls = []
        for _ in range(5):
            x, t = wall(lambda: eng.run_circuit(c, prec))
            walls.append(t)
            eng.release(x)
        walls.sort()
        info = plan.passes()
        print(f"[{os.environ.get('PLAN_OPTS', '')}] n={n} {prec.value}: plan {t_plan0:.2f} / cached {t_plan1:.2f} ms, init {t_init:.2f}, execute "
              f"{t_exec:.2f} / {t_exec2:.2f}, release {t_rel:.2f}, run_circuit median {walls[2]:.2f} ms; "
              f"passes {plan.num_passes}: " +
              " ".join(f"{t:.2f}({i['num_gates']}g,{i['kernel']},{i['num_phases']}ph,L{i['low_bits']})"
                       for t, i in zip(per, info)), flush=True)
