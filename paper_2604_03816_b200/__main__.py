"""``python -m paper_2604_03816_b200`` -- the reference CLI's ``run``,
``bench-scaling`` and ``bench-fusion`` subcommands (ref
``pkg/src/aqsim/cli.py:194-381``) for the B200 engine.

Differences from ``aqsim run``: no memory governor / CPU fallback (the north
star removes it; the device refuses with ``AllocationError`` instead), and
``--verify`` needs the reference package (it compares against
``aqsim``'s ReferenceEngine, as ``cli.py:276-278`` does).
"""
from __future__ import annotations

import argparse
import json
import statistics
import sys
import time

from . import B200Engine, Precision, fuse, select_precision
from . import generators as gen
from .fusion import depth


def _load(spec: str, seed: int):
    """Builtin generator spec (ref generators.py:111-138 plus layered-N) or a
    QASM/JSON file through the reference parser when available."""
    parts = spec.lower().split("-")
    try:
        if parts[0] == "ghz" and len(parts) == 2:
            return gen.ghz_circuit(int(parts[1]))
        if parts[0] == "qft" and len(parts) == 2:
            return gen.qft_circuit(int(parts[1]))
        if parts[0] == "random" and len(parts) in (2, 3):
            n = int(parts[1])
            return gen.random_su2_circuit(n, int(parts[2]) if len(parts) == 3 else 20 * n, seed)
        if parts[0] == "layered" and len(parts) in (2, 3):
            return gen.layered_circuit(int(parts[1]), int(parts[2]) if len(parts) == 3 else 14, seed)
    except ValueError as exc:
        raise ValueError(f"bad generator spec {spec!r}: {exc}") from None
    try:
        from aqsim import qasm  # type: ignore
    except Exception:
        raise ValueError(f"unknown spec {spec!r} (QASM/JSON files need the aqsim parser)") from None
    try:
        with open(spec) as fh:
            return qasm.parse(fh.read())
    except OSError as exc:
        raise ValueError(str(exc)) from None


def cmd_run(args) -> int:
    t = {k: 0.0 for k in ("parse", "fuse", "precision", "select", "execute", "sample")}
    t0 = time.perf_counter()
    circuit = _load(args.circuit, args.seed)
    t["parse"] = time.perf_counter() - t0
    d0 = depth(circuit)
    if args.no_fuse:
        fused, d1 = circuit, d0
    else:
        t0 = time.perf_counter()
        fused, rep = fuse(circuit, args.fuse_width)
        t["fuse"] = time.perf_counter() - t0
        d1 = rep.fused_depth
    t0 = time.perf_counter()
    if args.precision == "auto":
        precision = select_precision(fused.num_qubits, len(fused.gates), args.precision_tol).chosen
    else:
        precision = Precision(args.precision)
    t["precision"] = time.perf_counter() - t0
    eng = B200Engine("b200-cli")
    t0 = time.perf_counter()
    state = eng.run_circuit(fused, precision)
    t["execute"] = time.perf_counter() - t0
    counts = None
    if args.shots > 0:
        t0 = time.perf_counter()
        counts = eng.sample(state, args.shots, args.seed).counts
        t["sample"] = time.perf_counter() - t0
    fidelity = None
    if args.verify:
        import aqsim  # type: ignore
        ref = aqsim.get_engine("reference").run_circuit(fused, aqsim.Precision(precision.value))
        fidelity = aqsim.state_fidelity(ref, state)
    if args.no_timing:
        t = {k: 0.0 for k in t}
    report = {"circuit_name": getattr(circuit, "name", "") or args.circuit, "n": circuit.num_qubits,
              "g_original": len(circuit.gates), "g_fused": len(fused.gates),
              "depth_before": d0, "depth_after": d1, "precision_chosen": precision.value,
              "engine_chosen": "b200", "wall_seconds": t, "fidelity_vs_reference": fidelity,
              "fallback_events": [], "counts": counts, "seed": args.seed}
    sys.stdout.write(json.dumps(report, indent=2, sort_keys=True) + "\n")
    return 0


def cmd_bench_scaling(args) -> int:
    """Paper Table-2 workload: random_su2_circuit(n, g*n, seed+n) (ref cli.py:304-337)."""
    eng = B200Engine("b200-cli")
    rows = []
    for n in (int(x) for x in args.qubits.split(",") if x):
        c = gen.random_su2_circuit(n, args.gates_per_qubit * n, args.seed + n)
        times = []
        for _ in range(args.repetitions):
            t0 = time.perf_counter()
            s = eng.run_circuit(c, Precision.DOUBLE)
            times.append(time.perf_counter() - t0)
            eng.release(s)
        med = 0.0 if args.no_timing else statistics.median(times)
        rows.append({"n": n, "gates": len(c.gates), "engine": "b200", "median_s": med})
    sys.stdout.write(json.dumps(rows, indent=2, sort_keys=True) + "\n")
    return 0


def cmd_noise_compare(args) -> int:
    """Exact outcome fidelity / TVD of depolarized Bell / GHZ circuits vs the
    ideal state (ref cli.py:384-417), density matrices evolved on the device
    (paper_2604_03816_b200.noise); JSON rows, exact columns only."""
    from . import noise
    eng = B200Engine("b200-cli")
    rows = []
    for width in (int(x) for x in args.widths.split(",") if x):
        circuit = gen.ghz_circuit(width)
        st = eng.run_circuit(circuit, Precision.DOUBLE)
        probs = st.probabilities()
        eng.release(st)
        ideal = {format(i, f"0{width}b"): float(q) for i, q in enumerate(probs)}
        for p in (float(x) for x in args.p_values.split(",") if x):
            rho = noise.evolve_noisy(circuit, p, engine=eng)
            f_cl, tvd = noise.metrics(noise.measure_distribution(rho), ideal)
            rows.append({"circuit": circuit.name, "width": width, "p": p,
                         "f_cl_exact": round(f_cl, 6), "tvd_exact": round(tvd, 6)})
    sys.stdout.write(json.dumps(rows, indent=2, sort_keys=True) + "\n")
    return 0


def cmd_bench_fusion(args) -> int:
    """Depth reduction and time of each circuit unfused vs fused (ref
    cli.py:340-381; JSON rows instead of the reference's table)."""
    eng = B200Engine("b200-cli")
    rows = []
    for spec in (s_.strip() for s_ in args.circuits.split(",") if s_.strip()):
        circuit = _load(spec, args.seed)
        fused, rep = fuse(circuit, args.fuse_width)

        def _median_run(target) -> float:
            times = []
            for _ in range(args.repetitions):
                t0 = time.perf_counter()
                s = eng.run_circuit(target, Precision.DOUBLE)
                times.append(time.perf_counter() - t0)
                eng.release(s)
            return statistics.median(times)

        if args.no_exec or args.no_timing:
            time_s = fused_time_s = 0.0
        else:
            time_s = _median_run(circuit)
            fused_time_s = _median_run(fused)
        rows.append({"circuit": getattr(circuit, "name", "") or spec, "original_depth": rep.original_depth,
                     "fused_depth": rep.fused_depth, "reduction_percent": round(rep.reduction_percent, 1),
                     "time_s": time_s, "fused_time_s": fused_time_s})
    sys.stdout.write(json.dumps(rows, indent=2, sort_keys=True) + "\n")
    return 0


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="python -m paper_2604_03816_b200")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run")
    r.add_argument("circuit")
    r.add_argument("--precision", default="auto", choices=["auto", "single", "double"])
    r.add_argument("--precision-tol", type=float, default=1e-4)
    r.add_argument("--fuse-width", type=int, default=2)
    r.add_argument("--no-fuse", action="store_true")
    r.add_argument("--shots", type=int, default=0)
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--verify", action="store_true")
    r.add_argument("--no-timing", action="store_true")
    b = sub.add_parser("bench-scaling")
    b.add_argument("--qubits", default="20,22,24,26,28")
    b.add_argument("--gates-per-qubit", type=int, default=10)
    b.add_argument("--repetitions", type=int, default=3)
    b.add_argument("--seed", type=int, default=0)
    b.add_argument("--no-timing", action="store_true")
    nz = sub.add_parser("noise-compare")
    nz.add_argument("--widths", default="2,3,4,5")
    nz.add_argument("--p-values", default="0.0,0.001,0.01")
    f = sub.add_parser("bench-fusion")
    f.add_argument("--circuits", default="qft-12,ghz-12,random-12")
    f.add_argument("--fuse-width", type=int, default=2)
    f.add_argument("--repetitions", type=int, default=3)
    f.add_argument("--seed", type=int, default=0)
    f.add_argument("--no-exec", action="store_true")
    f.add_argument("--no-timing", action="store_true")
    args = ap.parse_args(argv)
    try:
        return {"run": cmd_run, "bench-scaling": cmd_bench_scaling, "bench-fusion": cmd_bench_fusion,
                "noise-compare": cmd_noise_compare}[args.cmd](args)
    except ValueError as exc:
        print(f"error: {exc}", file=sys.stderr)
        return 2


if __name__ == "__main__":
    sys.exit(main())
