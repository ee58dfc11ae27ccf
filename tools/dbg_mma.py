import sys, time
import numpy as np
sys.path.insert(0, ".")
from oracle import sv_oracle as orc
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.b200 import B200Engine, plan_options
from paper_2604_03816_b200.circuit import Precision
from paper_2604_03816_b200.fusion import fuse
n = int(sys.argv[1]) if len(sys.argv) > 1 else 14
c = fuse(gen.layered_circuit(n, layers=6, seed=1), 2)[0]
e = B200Engine("dbg", options=plan_options(tensor_cores=2))
plan = e.plan(c, Precision.SINGLE)
print("passes", plan.num_passes, [plan.native.pass_info(p)["num_tc"] for p in range(plan.num_passes)], flush=True)
t0 = time.time()
got = e.run_circuit(c, Precision.SINGLE).amplitudes
print("ran in", time.time() - t0, flush=True)
want = orc.run_circuit(c, "single")
print("max abs", np.abs(got - want).max(), "norm", np.vdot(got, got).real, flush=True)
