"""Device time of every pass of a BASELINE workload, with the pass shape.
usage: python tools/pass_probe.py qft30|layered28|layered30|layered33 [reps]
(env PLAN_OPTS="streams=4,..." for planner options; SVB_REG_STAGES etc. pass through)"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_03816_b200 import B200Engine, Precision, fuse  # noqa: E402
from paper_2604_03816_b200 import generators as gen  # noqa: E402
from paper_2604_03816_b200.b200 import plan_options  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "qft30"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
kind, n = ("qft", int(name[3:])) if name.startswith("qft") else ("layered", int(name[7:]))
prec = Precision.SINGLE if name == "layered28" else Precision.DOUBLE
c = gen.qft_circuit(n) if kind == "qft" else gen.layered_circuit(n)
f, _ = fuse(c, 2)
opts = {k: float(v) if "." in v else int(v) for k, v in
        (kv.split("=") for kv in os.environ.get("PLAN_OPTS", "").split(",") if kv)}
eng = B200Engine("probe", options=plan_options(**opts) if opts else None)
plan = eng.plan(f, prec)
st = eng.init_state(n, prec)
s = eng.stream()
plan.execute(st.tensor, s)
torch.cuda.synchronize()
per = [0.0] * plan.num_passes
for _ in range(reps):
    for p in range(plan.num_passes):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        plan.execute(st.tensor, s, p, 1)
        torch.cuda.synchronize()
        per[p] += (time.perf_counter() - t0) * 1e3 / reps
info = plan.passes()
hbm = 2 * (1 << n) * (8 if prec == Precision.SINGLE else 16) / 6445e9 * 1e3
print(f"{name} [{os.environ.get('PLAN_OPTS', '')}] total {sum(per):.2f} ms, HBM floor {hbm:.2f} ms/pass")
for p, (t, i) in enumerate(zip(per, info)):
    ops = [plan.native.kernel_op(p, k)["kind"][:2] + str(plan.native.kernel_op(p, k)["k"])
           for k in range(i["num_kernel_ops"])]
    print(f"  pass {p}: {t:7.2f} ms ({hbm / t:4.2f} HBM) {i['kernel']} L{i['low_bits']} high{i['high']} "
          f"gates {i['num_gates']} phases {i['num_phases']} streams {i['streams']} ops {' '.join(ops)}")
