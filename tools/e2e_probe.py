import sys, time
sys.path.insert(0, ".")
import torch
from paper_2604_03816_b200 import B200Engine
from paper_2604_03816_b200 import generators as gen
from paper_2604_03816_b200.fusion import fuse
from paper_2604_03816_b200.circuit import Precision
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
f, _ = fuse(gen.layered_circuit(n), 2)
eng = B200Engine("e2e")
for k in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan = eng.plan(f, Precision.DOUBLE)
    t1 = time.perf_counter()
    st = eng.init_state(n, Precision.DOUBLE)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    eng.execute(st, plan)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    nrm = eng.norm_squared(st)
    a0 = complex(st.tensor[0].item())
    t4 = time.perf_counter()
    eng.release(st)
    del st
    print(f"plan {1e3*(t1-t0):.1f} ms init {1e3*(t2-t1):.1f} exec {1e3*(t3-t2):.1f} read {1e3*(t4-t3):.1f}", flush=True)
