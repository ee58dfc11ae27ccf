#!/usr/bin/env python
"""Benchmark of the B200 state-vector engine (BASELINE.json metric: gates/s and
circuit time, % of the HBM roofline).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config layered28|qft30|layered33|layered-N|qft-N] [--precision single|double]

One *step* = one full circuit: |0...0> preparation plus every planned pass of
the fused circuit, inputs (the state) resident in HBM.  The default N=1
workload is BASELINE config 2: the seeded 28-qubit layered circuit (973 gates,
fused to 189 at width 2) in complex64.  ``value`` counts ORIGINAL (unfused)
gates per second.  The same JSON line carries ``configs``: BASELINE configs 3
(qft-30 c128) and 4 (layered-33 c128, 128 GiB) measured in the same run.  For
N>1 the state is sharded over the ranks (top log2 N qubits global) -- weak
scaling on the north star's sharded curve: n = 33 + log2 N c64 (N = 8 is
BASELINE config 5, 36 qubits), with the NVLink fraction of the swaps against
a peer bandwidth measured in the same run.

``--impl reference`` times the reference's NumPy algorithm (the oracle port in
oracle/, single-threaded like ref engines.py:190-203) on a bounded sample of the
same workload: each step applies the next fused gate of the circuit at full n.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# sizeof(svb::PassArgs<C>) (csrc/svb_types.h): header 64 B + 48 ops x 80 B + 24 KiB pool
PASS_ARGS_BYTES = 64 + 48 * 80 + 24576


def parse_args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--config", default=None)
    ap.add_argument("--precision", default=None, choices=[None, "single", "double"])
    ap.add_argument("--fuse-width", type=int, default=2)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cost-budget", type=float, default=0.0)
    ap.add_argument("--stages", type=int, default=0)
    ap.add_argument("--tile-bits", type=int, default=0)
    ap.add_argument("--min-low-bits", type=int, default=0)
    ap.add_argument("--reg-bits", type=int, default=0)
    ap.add_argument("--no-reg-phases", action="store_true")
    ap.add_argument("--pass-times", action="store_true", help="print per-pass device times to stderr")
    ap.add_argument("--tensor-cores", type=int, default=0, help="1 on, -1 off, 0 default")
    ap.add_argument("--tc-min-dense", type=int, default=0)
    ap.add_argument("--streams", type=int, default=0, help="tile streams per CTA (0 default)")
    ap.add_argument("--gemm-warps", type=int, default=0, help="k_gemm_pass warps per tile stream (4/8)")
    ap.add_argument("--no-configs", action="store_true",
                    help="skip the other single-GPU BASELINE configs (qft-30 / layered-33 c128)")
    ap.add_argument("--config-steps", type=int, default=3, help="timed steps of each extra config")
    return ap.parse_args()


def workload(args, world: int):
    """(name, circuit, precision) for the configuration."""
    from paper_2604_03816_b200 import generators as gen
    from paper_2604_03816_b200.precision import select_precision

    extra = int(round(math.log2(world))) if world > 1 else 0
    cfg = args.config or "layered28"
    if cfg == "layered28":
        # N = 1: BASELINE config 2 (28 q); N > 1: the north star's sharded
        # curve, 33 + log2 N qubits c64 (N = 8 is config 5, 36 q)
        n, kind, prec = (28 if world == 1 else 33 + extra), "layered", "single"
    elif cfg == "qft30":
        n, kind, prec = 30 + extra, "qft", "double"
    elif cfg == "layered33":
        n, kind, prec = 33 + extra, "layered", "double"
    elif cfg.startswith("layered-"):
        n, kind, prec = int(cfg.split("-")[1]), "layered", "single"
    elif cfg.startswith("qft-"):
        n, kind, prec = int(cfg.split("-")[1]), "qft", "double"
    else:
        raise SystemExit(f"unknown config {cfg}")
    if args.precision:
        prec = args.precision
    circuit = gen.layered_circuit(n) if kind == "layered" else gen.qft_circuit(n)
    return cfg, kind, n, circuit, prec


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[3:7]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def plan_kernels(plan) -> str:
    """Kernel(s) the plan launches."""
    names = set()
    for p in range(plan.num_passes):
        info = plan.native.pass_info(p)
        tb = info["tile_bits"] - info["reg_bits"]
        if info["kernel"] == "gemm":
            names.add(f"k_gemm_pass<{info['streams']}>+tcgen05")
        elif info["kernel"] == "reg_tc":
            names.add(f"k_reg_pass<RB={info['reg_bits']},TB={tb}>+" + ("tcgen05" if tb == 7 else "mma.sync"))
        elif info["kernel"] == "reg":
            names.add(f"k_reg_pass<RB={info['reg_bits']},TB={tb}>")
        else:
            names.add("k_tile_pass")
    return "+".join(sorted(names))


def gate_flops_per_amp(fused):
    """Algorithmic real flops per amplitude of a fused circuit: a row of a
    gate with r non-zeros costs r complex multiplies and r-1 complex adds
    (8r - 2 flops; 6 for a diagonal, 8*2^k - 2 for a dense k-qubit gate)."""
    from paper_2604_03816_b200.circuit import effective_unitary as _eu
    total = 0
    for op in fused.gates:
        u = _eu(op)
        r = np.count_nonzero(u) / u.shape[0]
        total += 8 * r - 2
    return total


def fma_peak_tflops(device, prec, sm_mhz):
    """Vector FMA peak: SMs x FMA/clk/SM (FP32 128, FP64 64) x 2 x SM clock."""
    import torch
    fma_per_clk = 128 if prec == "single" else 64
    sms = torch.cuda.get_device_properties(device).multi_processor_count
    return sms * fma_per_clk * 2 * sm_mhz * 1e6 / 1e12


def compute_roofline(fused, n, pass_ms, peak_tflops):
    """FP64 (c128 configs) compute roofline: the gates' algorithmic flops
    over the summed pass time vs the vector FMA peak. c128 passes of layered
    circuits are bound here rather than by HBM."""
    fa = gate_flops_per_amp(fused)
    ach = fa * (1 << n) / (sum(pass_ms) / 1e3) / 1e12
    return {"bound": "fp64-fma", "achieved": ach, "peak": peak_tflops, "unit": "TFLOP/s",
            "frac": ach / peak_tflops, "flops_per_amp": fa,
            "floor_ms": fa * (1 << n) / (peak_tflops * 1e12) * 1e3,
            "note": "algorithmic flops of the fused gates (8 per complex MAC over each row's "
                    "non-zeros) vs SMs x 64 DFMA/clk x 2 x max SM clock; the kernel merges runs of "
                    "diagonal gates into one table multiply, so diagonal-heavy circuits (QFT) execute "
                    "fewer flops than counted"}


def tensor_flops(plan, n: int) -> float:
    """Tensor-core flops of one plan execution: each GEMM phase multiplies every
    amplitude's 64-real row by a 64 x 64 real block in three fp16 products
    (hi.hi + lo.hi + hi.lo): 3 x 2 x 64 x 2 flops per complex amplitude."""
    gemms = sum(plan.native.pass_info(p)["num_tc"] for p in range(plan.num_passes))
    return gemms * float(1 << n) * 3 * 2 * 64 * 2


def measured_traffic(cfg: str, prec: str, n: int):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the
    dominant kernel from the committed ncu --set full capture of this workload
    (profiles/traffic.json), or None when no capture exists."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as fh:
            ent = json.load(fh).get(f"{cfg}:{prec}:{n}")
        return None if ent is None else ent["bytes_per_launch"]
    except Exception:
        return None


def measured_peak_hbm():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


def measured_peak_tensor():
    """Dense fp16/bf16 tensor-core peak (MEASURED_PEAKS.json burst figure: a
    pass is a short kernel), else the profiling recipe's nominal 2250."""
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as fh:
            return float(json.load(fh)["bf16_tflops"]), "measured"
    except Exception:
        return 2250.0, "fallback"


def cpu_baseline(circuit_fused, g0: int, n: int, prec: str, budget_s: float = 20.0) -> dict:
    """Oracle (numpy restatement of ref engines.py kernels, 1 thread) on a
    bounded sample: consecutive fused gates at full n until ``budget_s``."""
    from concurrent.futures import ThreadPoolExecutor

    from oracle import sv_oracle as orc
    workers = os.cpu_count() or 1
    t0 = time.perf_counter()
    amps = orc.init_state(n, prec)
    t_init = time.perf_counter() - t0
    done = 0
    with ThreadPoolExecutor(workers) as pool:
        t0 = time.perf_counter()
        while done < len(circuit_fused.gates):
            orc.apply_gate_parallel(amps, n, circuit_fused.gates[done], pool, workers)
            done += 1
            if time.perf_counter() - t0 >= budget_s:
                break
        dt = time.perf_counter() - t0
    per_fused = g0 / len(circuit_fused.gates)
    return {"value": done * per_fused / dt, "unit": "gates/s", "cores": workers, "kind": "port",
            "sample": f"first {done} of {len(circuit_fused.gates)} fused gates at n={n} {prec} "
                      f"({dt:.1f} s, +{t_init:.1f} s init), reference kernels chunked over "
                      f"{workers} threads (ref ParallelEngine generalised); gates/s counts original "
                      f"gates ({per_fused:.3f} per fused gate)"}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return 0
    from concurrent.futures import ThreadPoolExecutor

    from oracle import sv_oracle as orc
    from paper_2604_03816_b200.fusion import fuse
    cfg, kind, n, circuit, prec = workload(args, world)
    fused, _ = fuse(circuit, args.fuse_width)
    g0, gf = len(circuit.gates), len(fused.gates)
    amps = orc.init_state(n, prec)
    times = []
    workers = os.cpu_count() or 1
    with ThreadPoolExecutor(workers) as pool:
        for step in range(args.warmup + args.steps):
            op = fused.gates[step % gf]
            t0 = time.perf_counter()
            orc.apply_gate_parallel(amps, n, op, pool, workers)
            dt = time.perf_counter() - t0
            if step >= args.warmup:
                times.append(dt)
    per_fused = g0 / gf
    total = sum(times)
    value = len(times) * per_fused / total
    line = {
        "impl": "reference", "metric": "gates/s", "value": value, "unit": "gates/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * total / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c64" if prec == "single" else "c128",
        "data": "synthetic seeded circuit",
        "config": {"workload": f"{cfg}: {kind}-{n} {prec}, fused {g0}->{gf} (width {args.fuse_width})",
                   "n_qubits": n, "g_original": g0, "g_fused": gf},
        "cpu_baseline": {"value": value, "unit": "gates/s", "cores": workers, "kind": "port",
                         "sample": f"one fused gate per step at full n={n} (oracle port of "
                                   "ref engines.py:62-105, chunked over all host threads as "
                                   "ref ParallelEngine engines.py:206-262); circuit time "
                                   f"extrapolates to {total / len(times) * gf:.1f} s"},
        "e2e": {"value": value, "unit": "gates/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


def run_b200(args):
    import torch
    import torch.distributed as dist

    from paper_2604_03816_b200 import B200Engine, plan_options
    from paper_2604_03816_b200.b200 import prec_code
    from paper_2604_03816_b200.fusion import fuse
    from paper_2604_03816_b200.precision import select_precision

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SVB_DIST_BACKEND=gloo: exercise the N>1 path with several ranks sharing
    # the devices of a smaller box (tests); NCCL over NVLink otherwise
    backend_name = os.environ.get("SVB_DIST_BACKEND", "nccl")
    if backend_name != "nccl":
        local %= torch.cuda.device_count()
    torch.cuda.set_device(local)
    if world > 1:
        if backend_name == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend_name)
    cfg, kind, n, circuit, prec = workload(args, world)
    fused, rep = fuse(circuit, args.fuse_width)
    g0, gf = len(circuit.gates), len(fused.gates)
    decision = select_precision(n, gf)
    from paper_2604_03816_b200.circuit import Precision
    precision = Precision(prec)
    opts = plan_options(cost_budget=args.cost_budget, stages=args.stages,
                        tile_bits=args.tile_bits, min_low_bits=args.min_low_bits,
                        reg_bits=args.reg_bits, no_reg_phases=int(args.no_reg_phases),
                        tensor_cores=args.tensor_cores, tc_min_dense=args.tc_min_dense,
                        streams=args.streams, gemm_warps=args.gemm_warps)
    eng = B200Engine("b200-bench", device=local, options=opts)

    if world > 1:
        return run_sharded(args, eng, fused, circuit, n, precision, cfg, kind, rank, world, local)

    m = measure(eng, fused, g0, n, precision, args.steps, args.warmup, args.pass_times)
    plan, n_passes, pass_ms, ms_step = m["plan"], m["n_passes"], m["pass_ms"], m["ms_step"]
    m_norm, m_clk = m["norm"], m["clocks"]
    value = g0 / (ms_step / 1e3)
    amp_bytes = precision.amplitude_bytes
    pc = prec_code(precision)
    state = m["state"]
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    peak, peak_kind = measured_peak_hbm()
    bytes_per_pass = 2 * (1 << n) * amp_bytes

    # single-gate pass (the north star's "per local gate pass"): one dense 2q
    # gate = one HBM round trip of the state with no compute to hide, timed
    # with CUDA events over 10 launches
    from paper_2604_03816_b200.circuit import Circuit as _Circ
    from paper_2604_03816_b200.circuit import GateKind as _GK
    from paper_2604_03816_b200.circuit import GateOp as _GO
    _rng = np.random.default_rng(5)
    _u, _ = np.linalg.qr(_rng.normal(size=(4, 4)) + 1j * _rng.normal(size=(4, 4)))
    gplan = eng.plan(_Circ(n, [_GO(_GK.CUSTOM, (3, n - 2), (), _u)]), precision)
    gplan.execute(state.tensor, s)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(10):
        gplan.execute(state.tensor, s)
    e1.record(stream)
    torch.cuda.synchronize()
    gate_ms = e0.elapsed_time(e1) / 10
    gate_pass = {"what": f"one dense 2q gate on qubits (3, {n - 2}) = one pass, 10 launches",
                 "ms": gate_ms, "achieved": bytes_per_pass / (gate_ms / 1e3) / 1e9,
                 "frac": bytes_per_pass / (gate_ms / 1e3) / 1e9 / peak}

    # e2e: public API from a host circuit: plan + launch (kernel-parameter H2D) +
    # run + device->host read of the result (norm^2 and amplitude 0).  Warm:
    # the content-keyed plan cache hits (the serving case); cold: a fresh
    # engine, so the native planner runs inside the timed region.
    eng.release(state)
    del state, m
    torch.cuda.empty_cache()
    h2d = n_passes * PASS_ARGS_BYTES  # __grid_constant__ parameter block per launch

    def e2e_once(engine):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = engine.run_circuit(fused, precision)
        engine.norm_squared(st)
        complex(st.tensor[0].item())
        dt = time.perf_counter() - t0
        engine.release(st)
        return dt

    e2e_times = []
    for k in range(max(2, min(args.steps, 5)) + 1):
        dt = e2e_once(eng)
        if k:
            e2e_times.append(dt)
    e2e_value = g0 / statistics.median(e2e_times)
    cold_times = [e2e_once(B200Engine("b200-cold", device=local, options=eng.options)) for _ in range(2)]
    torch.cuda.empty_cache()

    # compute rooflines of the same launches: algorithmic flops of the fused
    # gates (dense k-qubit: 8*2^k - 2 real flops per amplitude, diagonal: 6)
    # against the vector FMA peak, and the tensor-core flops the GEMM phases
    # issue against the measured dense fp16 peak
    flops_amp = gate_flops_per_amp(fused)
    sm_mhz = (m_clk or {}).get("sm_max_mhz") or 1965.0
    peak_tflops = fma_peak_tflops(local, prec, sm_mhz)
    achieved_tflops = flops_amp * (1 << n) / (sum(pass_ms) / 1e3) / 1e12
    tc_flops = tensor_flops(plan, n)
    tpeak, tpeak_kind = measured_peak_tensor()
    traffic = measured_traffic(cfg, prec, n)
    avg_pass_ms = sum(pass_ms) / n_passes
    achieved = bytes_per_pass / (avg_pass_ms / 1e3) / 1e9
    best_pass = min(pass_ms)

    # the other single-GPU BASELINE configs (3: qft-30 c128, 4: layered-33 c128)
    configs = {}
    if cfg == "layered28" and not args.no_configs:
        for name, circ, pr in (("qft30_c128", gen_circuit("qft", 30), "double"),
                               ("layered33_c128", gen_circuit("layered", 33), "double")):
            f2, _ = fuse(circ, args.fuse_width)
            ng0 = len(circ.gates)
            mm = measure(B200Engine("b200-cfg", device=local, options=eng.options), f2, ng0, circ.num_qubits,
                         Precision(pr), args.config_steps, 3, False)
            b2 = 2 * (1 << circ.num_qubits) * Precision(pr).amplitude_bytes
            apm = sum(mm["pass_ms"]) / mm["n_passes"]
            configs[name] = {"workload": f"{circ.name} {pr}, fused {ng0}->{len(f2.gates)}",
                             "value": ng0 / (mm["ms_step"] / 1e3), "unit": "gates/s",
                             "ms_per_step": mm["ms_step"], "steps": args.config_steps, "warmup": 3,
                             "passes": mm["n_passes"], "kernel": plan_kernels(mm["plan"]),
                             "roofline": {"bound": "hbm", "achieved": b2 / (apm / 1e3) / 1e9, "peak": peak,
                                          "unit": "GB/s", "frac": b2 / (apm / 1e3) / 1e9 / peak,
                                          "peak_kind": peak_kind, "avg_launch_ms": apm,
                                          "traffic": measured_traffic(name.split("_")[0], pr, circ.num_qubits)},
                             "compute": compute_roofline(f2, circ.num_qubits, mm["pass_ms"],
                                                         fma_peak_tflops(local, pr, sm_mhz)),
                             "norm_after": mm["norm"], "clocks": mm["clocks"]}
            eng_state = mm.pop("state")
            del eng_state, mm
            torch.cuda.empty_cache()

    cpu = None
    if not args.no_cpu_baseline:
        torch.cuda.empty_cache()
        cpu = cpu_baseline(fused, g0, n, prec, budget_s=20.0)

    line = {
        "metric": "gates/s", "value": value, "unit": "gates/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "c64" if prec == "single" else "c128", "data": "synthetic seeded circuit",
        "config": {"workload": f"{cfg}: {kind}-{n} {prec}, fused {g0}->{gf} (width {args.fuse_width})",
                   "n_qubits": n, "g_original": g0, "g_fused": gf, "passes": n_passes,
                   "state_bytes": (1 << n) * amp_bytes,
                   "l2": "state larger than the 126 MB L2; no flush needed",
                   "precision_decision": decision.rationale + " (bench forces "
                   + prec + " as BASELINE config names it)",
                   "circuit_ms": ms_step, "fused_gates_per_s": gf / (ms_step / 1e3),
                   "passes_per_s": n_passes / (ms_step / 1e3), "norm_after": m_norm},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                     "kernel": plan_kernels(plan), "bytes_per_launch": bytes_per_pass,
                     "avg_launch_ms": avg_pass_ms, "best_launch_ms": best_pass,
                     "best_frac": bytes_per_pass / (best_pass / 1e3) / 1e9 / peak,
                     "pass_ms": [round(x, 4) for x in pass_ms],
                     "single_gate_pass": gate_pass,
                     "tensor": {"achieved": tc_flops / (sum(pass_ms) / 1e3) / 1e12, "peak": tpeak,
                                "unit": "TFLOP/s", "peak_kind": tpeak_kind,
                                "frac": tc_flops / (sum(pass_ms) / 1e3) / 1e12 / tpeak,
                                "flops_per_step": tc_flops,
                                "note": "fp16 tcgen05 GEMM phases: 3 products (hi.hi, lo.hi, hi.lo) of a "
                                        "64x64 real block per amplitude row"},
                     # the pipe that executes the gate arithmetic: tcgen05 (fp16 hi/lo
                     # products) when the plan runs GEMM phases, else the vector FMA pipe
                     "compute": ({"bound": "tensor-fp16", "pipe": "tcgen05.mma kind::f16",
                                  "achieved": tc_flops / (sum(pass_ms) / 1e3) / 1e12, "peak": tpeak,
                                  "unit": "TFLOP/s", "peak_kind": tpeak_kind,
                                  "frac": tc_flops / (sum(pass_ms) / 1e3) / 1e12 / tpeak,
                                  "note": "GEMM-phase tensor flops (roofline.tensor); the gates' "
                                          "algorithmic flops vs the FP32 FMA peak are in "
                                          "compute_vector_reference"}
                                 if tc_flops > 0 else
                                 {"bound": "fp32-fma" if prec == "single" else "fp64-fma",
                                  "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                                  "frac": achieved_tflops / peak_tflops, "flops_per_amp": flops_amp,
                                  "note": "algorithmic gate flops vs the vector FMA peak (SMs x FMA/clk "
                                          "x 2 x max SM clock)"}),
                     "compute_vector_reference": {
                         "bound": "fp32-fma" if prec == "single" else "fp64-fma",
                         "achieved": achieved_tflops, "peak": peak_tflops, "unit": "TFLOP/s",
                         "frac": achieved_tflops / peak_tflops, "flops_per_amp": flops_amp,
                         "note": "algorithmic gate flops vs the vector FMA peak; above 1 when the "
                                 "phases run on the tensor cores instead"}},
        "configs": configs,
        "e2e": {"value": e2e_value, "unit": "gates/s", "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": 8 + (8 if pc == 0 else 16),
                "path": "B200Engine.run_circuit(fused circuit; plan cached by content after the first, "
                        "untimed call) + norm_squared + amplitude[0] read",
                "cold": {"value": g0 / statistics.median(cold_times), "unit": "gates/s",
                         "path": "same call on a fresh engine: native planning inside the timed region"}},
        "gpu_launches": args.steps * (n_passes + 2),
        "clocks": m_clk,
        "cpu_baseline": cpu,
    }
    print(json.dumps(line))
    return 0


def gen_circuit(kind: str, n: int):
    from paper_2604_03816_b200 import generators as gen
    return gen.layered_circuit(n) if kind == "layered" else gen.qft_circuit(n)


def measure(eng, fused, g0: int, n: int, precision, steps: int, warmup: int, pass_times: bool = False) -> dict:
    """Device time of `steps` circuit executions (|0> preparation + every pass),
    CUDA events around the whole timed region and around each pass, clocks
    sampled during it."""
    import ctypes as C

    import torch

    from paper_2604_03816_b200 import _native
    from paper_2604_03816_b200.b200 import prec_code
    plan = eng.plan(fused, precision)
    n_passes = plan.num_passes
    state = eng.init_state(n, precision)
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    L = _native.lib()
    pc = prec_code(precision)

    def step(events=None):
        _native.check(L.svb_fill_basis(C.c_void_p(state.tensor.data_ptr()), n, pc, 0, C.c_void_p(s)))
        if events is None:
            plan.execute(state.tensor, s)
        else:
            for p in range(n_passes):
                events[p][0].record(stream)
                plan.execute(state.tensor, s, p, 1)
                events[p][1].record(stream)

    for _ in range(warmup):
        step()
    torch.cuda.synchronize()
    ev = [[(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(n_passes)] for _ in range(steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(torch.cuda.current_device()) as clk:
        torch.cuda.synchronize()
        start.record(stream)
        for k in range(steps):
            step(ev[k])
        stop.record(stream)
        torch.cuda.synchronize()
    total_ms = start.elapsed_time(stop)
    pass_ms = [sum(ev[k][p][0].elapsed_time(ev[k][p][1]) for k in range(steps)) / steps
               for p in range(n_passes)]
    if pass_times:
        for p_, ms_ in enumerate(pass_ms):
            info = plan.native.pass_info(p_)
            ops = [plan.native.kernel_op(p_, i)["kind"][0] + str(plan.native.kernel_op(p_, i)["k"])
                   for i in range(info["num_kernel_ops"])]
            fl = [plan.native.phase(p_, f)["flags"] for f in range(info["num_phases"])]
            print(f"pass {p_:3d} {ms_:.3f} ms frac {2 * (1 << n) * precision.amplitude_bytes / ms_ / 1e6 / 6445:.2f} "
                  f"{info['kernel']} L={info['low_bits']} high={info['high']} phases={info['num_phases']} "
                  f"gemms={info['num_tc']} flags={fl} conf={info['bank_conflicts']} ops={ops}", file=sys.stderr)
    return {"plan": plan, "n_passes": n_passes, "pass_ms": pass_ms, "ms_step": total_ms / steps,
            "state": state, "norm": eng.norm_squared(state), "clocks": clk.summary()}


def p2p_peak_gbs(dist, red_dev, local) -> float:
    """Peer bandwidth per direction measured here: every rank sends 1 GiB to and
    receives 1 GiB from rank ^ 1 (NCCL over NVLink), best of 3, min over ranks."""
    import torch
    rank, world = dist.get_rank(), dist.get_world_size()
    peer = rank ^ 1
    if peer >= world:
        return None
    a = torch.empty(1 << 27, dtype=torch.float64, device=f"cuda:{local}")
    b = torch.empty_like(a)
    best = 0.0
    for _ in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in dist.batch_isend_irecv([dist.P2POp(dist.isend, a, peer), dist.P2POp(dist.irecv, b, peer)]):
            r.wait()
        e1.record()
        torch.cuda.synchronize()
        best = max(best, a.numel() * 8 / (e0.elapsed_time(e1) / 1e3) / 1e9)
    t = torch.tensor([best], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t, op=dist.ReduceOp.MIN)
    del a, b
    torch.cuda.empty_cache()
    return float(t.item())


def run_sharded(args, eng, fused, circuit, n, precision, cfg, kind, rank, world, local):
    """N>1: state sharded over the ranks (top log2 N qubits global), NCCL swaps."""
    import torch
    import torch.distributed as dist

    from paper_2604_03816_b200.sharded import CudaShardBackend, ShardedEngine, SwapStep

    red_dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo reduces host tensors
    backend = CudaShardBackend(local, eng.options)
    sh = ShardedEngine(backend)
    sched, progs = sh.compile(fused, precision)
    n_local = sched.n_local
    g0, gf = len(circuit.gates), len(fused.gates)
    state = sh.init_state(n_local, precision)
    stream = torch.cuda.current_stream()
    amp_bytes = precision.amplitude_bytes
    n_passes = sum(p.num_passes for k, p in progs if k == "local")
    swaps = [p for k, p in progs if k == "swap"]

    def step(ev=None):
        backend.fill(state, 0 if rank == 0 else -1)
        for kind_, obj in progs:
            if ev is not None:
                ev.append((kind_, torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)))
                ev[-1][1].record(stream)
            if kind_ == "local":
                backend.run(state, obj)
            else:
                sh.exchange(state, obj)
            if ev is not None:
                ev[-1][2].record(stream)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    evs = [[] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        dist.barrier()
        torch.cuda.synchronize()
        start.record(stream)
        for k in range(args.steps):
            step(evs[k])
        stop.record(stream)
        torch.cuda.synchronize()
        dist.barrier()
    t_ms = torch.tensor([start.elapsed_time(stop)], dtype=torch.float64, device=red_dev)
    dist.all_reduce(t_ms, op=dist.ReduceOp.MAX)
    ms_step = float(t_ms.item()) / args.steps
    local_ms = sum(a.elapsed_time(b) for e in evs for k_, a, b in e if k_ == "local") / args.steps
    swap_ms = sum(a.elapsed_time(b) for e in evs for k_, a, b in e if k_ == "swap") / args.steps
    agg = torch.tensor([local_ms, swap_ms], dtype=torch.float64, device=red_dev)
    dist.all_reduce(agg, op=dist.ReduceOp.MAX)
    local_ms, swap_ms = (float(x) for x in agg.tolist())
    norm = backend.norm2(state)
    nt = torch.tensor([norm], dtype=torch.float64, device=red_dev)
    dist.all_reduce(nt)
    bytes_per_pass = 2 * (1 << n_local) * amp_bytes
    peak, peak_kind = measured_peak_hbm()
    achieved = bytes_per_pass * n_passes / (local_ms / 1e3) / 1e9 if n_passes else 0.0
    sent = sum((1 - 2.0 ** -s_.m) * (1 << n_local) * amp_bytes for s_ in swaps)
    nvl = sent / (swap_ms / 1e3) / 1e9 if swap_ms > 0 else None
    nvl_peak = p2p_peak_gbs(dist, red_dev, local) if dist.get_backend() == "nccl" else None
    # e2e through the public sharded API (schedule + plan + run + all-reduced norm)
    e2e = []
    for k in range(3):
        torch.cuda.synchronize()
        dist.barrier()
        t0 = time.perf_counter()
        st = sh.run_circuit(fused, precision)
        _ = st.norm_squared()
        dt = torch.tensor([time.perf_counter() - t0], dtype=torch.float64, device=red_dev)
        dist.all_reduce(dt, op=dist.ReduceOp.MAX)
        if k:
            e2e.append(float(dt.item()))
        del st
        torch.cuda.empty_cache()
    if rank == 0:
        line = {
            "metric": "gates/s", "value": g0 / (ms_step / 1e3), "unit": "gates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "c64" if precision.value == "single" else "c128", "data": "synthetic seeded circuit",
            "config": {"workload": f"{cfg}: {kind}-{n} {precision.value}, fused {g0}->{gf}, sharded "
                                   f"{world} ranks (n_local {n_local})",
                       "n_qubits": n, "n_local": n_local, "g_original": g0, "g_fused": gf,
                       "passes_per_rank": n_passes, "swaps": len(swaps),
                       "parallelism": f"state sharded over {world} GPUs (top {sched.g} qubits global)",
                       "l2": "shard larger than L2", "local_ms": local_ms, "swap_ms": swap_ms,
                       "norm_after": float(nt.item())},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": None, "peak_kind": peak_kind,
                         "kernel": "local passes (k_gemm_pass / k_reg_pass); swaps: k_swap over CUDA-IPC peer memory"
                                   if sh._use_p2p(backend.tensor(state)) else "local passes; swaps: NCCL send/recv",
                         "nvlink": {"bytes_sent_per_gpu": sent, "achieved_gbs": nvl,
                                    "peak_gbs": nvl_peak,
                                    "peak_kind": "measured: 1 GiB pairwise send/recv, max over ranks",
                                    "frac": (nvl / nvl_peak) if (nvl and nvl_peak) else None}},
            "e2e": {"value": g0 / statistics.median(e2e), "unit": "gates/s",
                    "h2d_bytes_per_step": n_passes * PASS_ARGS_BYTES, "d2h_bytes_per_step": 8},
            # passes + the |0> fill (2 kernels) + one swap kernel per swap (p2p)
            "gpu_launches": args.steps * (n_passes + 2 + (len(swaps) if sh._use_p2p(backend.tensor(state)) else 0)),
            "clocks": clk.summary(),
            "cpu_baseline": None,
        }
        print(json.dumps(line))
    dist.destroy_process_group()
    return 0


def main():
    args = parse_args()
    if args.impl == "reference":
        return run_reference(args)
    return run_b200(args)


if __name__ == "__main__":
    sys.exit(main())
