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
st = eng.run_circuit(f, Precision.DOUBLE)
for k in range(6):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    nrm = eng.norm_squared(st)
    t1 = time.perf_counter()
    a0 = complex(st.tensor[0].item())
    t2 = time.perf_counter()
    print(f"norm {1e3*(t1-t0):.1f} ms item {1e3*(t2-t1):.1f} ms", flush=True)
for k in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    eng.execute(st, eng.plan(f, Precision.DOUBLE))
    t1 = time.perf_counter()
    nrm = eng.norm_squared(st)
    t2 = time.perf_counter()
    print(f"exec-enqueue {1e3*(t1-t0):.1f} ms norm(after exec) {1e3*(t2-t1):.1f} ms", flush=True)
