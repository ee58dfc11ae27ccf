"""Stage timeline of one k_gemm_pass launch (CTA 0, tile stream 0): run with
SVB_GEMM_TRACE=1.  usage: SVB_GEMM_TRACE=1 python tools/gemm_trace.py [pass]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2604_03816_b200 import B200Engine, Precision, fuse  # noqa: E402
from paper_2604_03816_b200 import _native  # noqa: E402
from paper_2604_03816_b200 import generators as gen  # noqa: E402

p = int(sys.argv[1]) if len(sys.argv) > 1 else 3
eng = B200Engine("trace")
f, _ = fuse(gen.layered_circuit(28), 2)
plan = eng.plan(f, Precision.SINGLE)
st = eng.init_state(28, Precision.SINGLE)
for _ in range(3):
    plan.execute(st.tensor, eng.stream())
plan.execute(st.tensor, eng.stream(), p, 1)
torch.cuda.synchronize()
buf = (C.c_ulonglong * 128)()
n = _native.lib().svb_debug_trace(buf, 128)
info = plan.native.pass_info(p)
print(f"pass {p}: {info['kernel']} gemms {info['num_tc']} (events: start, landed, loaded+norm, A1 written, "
      f"[GEMM done, A written]..., GEMM P done, out-norm, stored)")
for t in range(8):
    ev = [buf[t * 16 + i] for i in range(16)]
    ev = [e for e in ev if e]
    if not ev:
        continue
    d = [ev[i + 1] - ev[i] for i in range(len(ev) - 1)]
    nxt = buf[(t + 1) * 16] - ev[0] if t < 7 and buf[(t + 1) * 16] else 0
    print(f"tile {t}: total {ev[-1] - ev[0]:6d} cyc  next-start {nxt:6d}  stages {d}")
