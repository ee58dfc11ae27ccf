"""Kernel-efficiency probe: passes whose gates all act on the same few qubits
(one register phase) vs. spread over the tile (many phases).  Prints the FMA
rate of each plan against the vector FMA peak."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2604_03816_b200 import B200Engine  # noqa: E402
from paper_2604_03816_b200.circuit import Circuit, GateKind, GateOp, Precision  # noqa: E402


def rand_u(k, rng):
    z = rng.normal(size=(1 << k, 1 << k)) + 1j * rng.normal(size=(1 << k, 1 << k))
    q, _ = np.linalg.qr(z)
    return q


def run(name, n, gates, prec, reps=5):
    eng = B200Engine("probe")
    c = Circuit(n, gates)
    plan = eng.plan(c, prec)
    st = eng.init_state(n, prec)
    s = torch.cuda.current_stream()
    for _ in range(2):
        plan.execute(st.tensor, s.cuda_stream)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        plan.execute(st.tensor, s.cuda_stream)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fma = sum(4 * (1 << len(g.targets)) for g in gates) * (1 << n)
    peak = 148 * (128 if prec is Precision.SINGLE else 64) * 1.965e9
    hbm = plan.num_passes * 2 * (1 << n) * prec.amplitude_bytes / 6.65e12 * 1e3
    infos = [plan.native.pass_info(p) for p in range(plan.num_passes)]
    print(f"{name:40s} {prec.name:6s} passes {plan.num_passes:2d} phases {sum(i['num_phases'] for i in infos):3d} "
          f"{ms:8.3f} ms  FMA {fma / ms / 1e-3 / peak:5.1%} of peak  (HBM floor {hbm:.2f} ms)", flush=True)
    eng.release(st)


def main():
    rng = np.random.default_rng(0)
    only = sys.argv[1] if len(sys.argv) > 1 else None
    for prec, n in ((Precision.SINGLE, 28), (Precision.DOUBLE, 28)):
        if only and only != prec.name:
            continue
        hi = 8 if prec is Precision.SINGLE else 6
        # one phase: 24 dense 2q gates on 4 qubits inside the register set
        g = [GateOp(GateKind.CUSTOM, (hi + (i % 3), hi + (i % 3) + 1), (), rand_u(2, rng)) for i in range(24)]
        run("1 phase, 24 x 2q on 4 qubits", n, g, prec)
        if only:
            return
        g = [GateOp(GateKind.CUSTOM, (hi + (i % 2) * 2, hi + (i % 2) * 2 + 1), (), rand_u(2, rng)) for i in range(24)]
        run("1 phase, 24 x 2q disjoint pairs", n, g, prec)
        g = [GateOp(GateKind.CUSTOM, (hi + 1,), (), rand_u(1, rng)) for i in range(48)]
        run("1 phase, 48 x 1q", n, g, prec)
        # brickwork over the low 12 qubits: several phases
        g = []
        for layer in range(8):
            for q in range(layer % 2, 11, 2):
                g.append(GateOp(GateKind.CUSTOM, (q, q + 1), (), rand_u(2, rng)))
        run("brickwork 12 qubits x 8 layers", n, g, prec)
        g = [GateOp(GateKind.CUSTOM, (2 * i % 12, 2 * i % 12 + 1), (), rand_u(2, rng)) for i in range(1)]
        run("1 gate (HBM pass)", n, g, prec)


if __name__ == "__main__":
    main()
