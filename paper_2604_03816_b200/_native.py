"""ctypes binding of libsvb200.so (the C ABI in include/svb200.h).

There is no fallback: if the shared library is missing or fails to load,
every entry point raises.  Planning calls (``plan_*``) are host-only and work
without a GPU; everything that touches amplitudes needs a CUDA device.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

# SVB_LIB: load another build of the library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("SVB_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libsvb200.so")

SVB_C64, SVB_C128 = 0, 1
SVB_OK, SVB_EINVAL, SVB_ECUDA, SVB_ENOMEM, SVB_EUNSUPPORTED = 0, -1, -2, -3, -4
SVB_MAX_TARGETS = 8
ABI_VERSION = 2

# every symbol declared in include/svb200.h (tests check the library exports them)
EXPORTS = (
    "svb_abi_version", "svb_debug_trace", "svb_last_error", "svb_device_sm_count", "svb_fill_basis",
    "svb_apply_gate", "svb_plan_create", "svb_plan_num_passes", "svb_plan_pass_info",
    "svb_plan_pass_gates", "svb_plan_kernel_op", "svb_plan_phase", "svb_plan_phase_op",
    "svb_plan_phase_tc", "svb_plan_tc_matrix", "svb_plan_phase_op_ext", "svb_plan_phase_map",
    "svb_plan_execute",
    "svb_plan_execute_range", "svb_plan_destroy", "svb_dot", "svb_dot_mixed", "svb_norm2",
    "svb_probabilities", "svb_block_sums", "svb_sample_search", "svb_swap_blocks",
    "svb_enable_peer_access", "svb_ipc_export", "svb_ipc_import", "svb_ipc_close",
)


class PlanOptions(C.Structure):
    _fields_ = [("tile_bits", C.c_int), ("min_low_bits", C.c_int),
                ("max_ops_per_pass", C.c_int), ("cost_budget", C.c_double),
                ("no_diag_merge", C.c_int), ("stages", C.c_int), ("reg_bits", C.c_int),
                ("no_reg_phases", C.c_int), ("tensor_cores", C.c_int), ("tc_min_dense", C.c_int),
                ("no_window_search", C.c_int), ("streams", C.c_int), ("gemm_warps", C.c_int),
                ("no_factor", C.c_int), ("no_gate_merge", C.c_int)]


class PassInfo(C.Structure):
    _fields_ = [("tile_bits", C.c_int), ("low_bits", C.c_int), ("num_high", C.c_int),
                ("high", C.c_int * 8), ("num_kernel_ops", C.c_int), ("num_gates", C.c_int),
                ("est_cost", C.c_double), ("reg_bits", C.c_int), ("num_phases", C.c_int),
                ("num_tc", C.c_int), ("kernel", C.c_int), ("streams", C.c_int),
                ("bank_conflicts", C.c_int)]


KERNELS = ("tile", "reg", "reg_tc", "gemm")
KINDS = ("dense", "diag", "perm", "ctrl")  # OpKind; "perm" = CNOT (control, target); "ctrl" = U0/U1 by a thread bit


class NativeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        self.code = code
        super().__init__(f"libsvb200 error {code}: {msg}")


_lib = None


def lib():
    """Load (once) and return the library; raises if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -m paper_2604_03816_b200._build` "
            "(the B200 engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    vp, i, ll, d = C.c_void_p, C.c_int, C.c_longlong, C.c_double
    ip, dp = C.POINTER(C.c_int), C.POINTER(C.c_double)
    sig = {
        "svb_abi_version": (i, []),
        "svb_debug_trace": (i, [C.POINTER(C.c_ulonglong), i]),
        "svb_last_error": (C.c_char_p, []),
        "svb_device_sm_count": (i, [ip]),
        "svb_fill_basis": (i, [vp, i, i, ll, vp]),
        "svb_apply_gate": (i, [vp, i, i, i, ip, dp, vp]),
        "svb_plan_create": (i, [i, i, i, ip, ip, dp, C.POINTER(PlanOptions), C.POINTER(vp)]),
        "svb_plan_num_passes": (i, [vp]),
        "svb_plan_pass_info": (i, [vp, i, C.POINTER(PassInfo)]),
        "svb_plan_pass_gates": (i, [vp, i, ip, i]),
        "svb_plan_kernel_op": (i, [vp, i, i, ip, ip, ip, dp, i]),
        "svb_plan_phase": (i, [vp, i, i, ip, ip, ip, ip]),
        "svb_plan_phase_op": (i, [vp, i, i, ip, ip, ip, ip, dp, i]),
        "svb_plan_phase_tc": (i, [vp, i, i, ip, ip]),
        "svb_plan_phase_op_ext": (i, [vp, i, i, ip, C.POINTER(C.c_ulonglong)]),
        "svb_plan_phase_map": (i, [vp, i, i, ip, ip]),
        "svb_plan_tc_matrix": (i, [vp, i, i, dp, i]),
        "svb_plan_execute": (i, [vp, vp, vp]),
        "svb_plan_execute_range": (i, [vp, vp, i, i, vp]),
        "svb_plan_destroy": (None, [vp]),
        "svb_dot": (i, [vp, vp, i, i, dp, vp]),
        "svb_dot_mixed": (i, [vp, i, vp, i, i, dp, vp]),
        "svb_norm2": (i, [vp, i, i, dp, vp]),
        "svb_probabilities": (i, [vp, i, ll, ll, vp, vp]),
        "svb_block_sums": (i, [vp, i, i, i, vp, vp]),
        "svb_sample_search": (i, [vp, i, i, i, vp, vp, ll, vp, vp]),
        "svb_swap_blocks": (i, [vp, vp, ll, vp]),
        "svb_enable_peer_access": (i, [i, i]),
        "svb_ipc_export": (i, [vp, vp, C.POINTER(C.c_longlong)]),
        "svb_ipc_import": (i, [vp, ll, C.POINTER(vp), C.POINTER(vp)]),
        "svb_ipc_close": (i, [vp]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    if L.svb_abi_version() != ABI_VERSION:
        raise RuntimeError(f"libsvb200 ABI {L.svb_abi_version()} != expected {ABI_VERSION}")
    _lib = L
    return L


def check(rc: int) -> int:
    if rc < 0:
        msg = lib().svb_last_error().decode(errors="replace")
        if rc == SVB_EINVAL:
            raise ValueError(msg)
        raise NativeError(rc, msg)
    return rc


def _iptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_int))


def _dptr(a: np.ndarray):
    return a.ctypes.data_as(C.POINTER(C.c_double))


class NativePlan:
    """Owns an ``svb_plan*``; host-side only until ``execute``."""

    def __init__(self, n_local: int, prec: int, ks: np.ndarray, targets: np.ndarray,
                 mats: np.ndarray, options: PlanOptions | None = None):
        self._h = None
        self.n_local = n_local
        self.prec = prec
        self.num_gates = int(ks.size)
        ks = np.ascontiguousarray(ks, dtype=np.int32)
        targets = np.ascontiguousarray(targets, dtype=np.int32)
        mats = np.ascontiguousarray(mats, dtype=np.float64)
        h = C.c_void_p()
        opt = C.byref(options) if options is not None else None
        check(lib().svb_plan_create(n_local, prec, int(ks.size), _iptr(ks), _iptr(targets),
                                    _dptr(mats), opt, C.byref(h)))
        self._h = h

    @property
    def handle(self):
        return self._h

    def num_passes(self) -> int:
        return check(lib().svb_plan_num_passes(self._h))

    def pass_info(self, p: int) -> dict:
        info = PassInfo()
        check(lib().svb_plan_pass_info(self._h, p, C.byref(info)))
        return {"tile_bits": info.tile_bits, "low_bits": info.low_bits,
                "high": [info.high[b] for b in range(info.num_high)],
                "num_kernel_ops": info.num_kernel_ops, "num_gates": info.num_gates,
                "est_cost": info.est_cost, "reg_bits": info.reg_bits, "num_phases": info.num_phases,
                "num_tc": info.num_tc, "kernel": KERNELS[info.kernel], "streams": info.streams,
                "bank_conflicts": info.bank_conflicts}

    def phase(self, p: int, f: int) -> dict:
        R = (C.c_int * 8)()
        b, e, fl = C.c_int(), C.c_int(), C.c_int()
        check(lib().svb_plan_phase(self._h, p, f, R, C.byref(b), C.byref(e), C.byref(fl)))
        mid, tc = C.c_int(), C.c_int()
        check(lib().svb_plan_phase_tc(self._h, p, f, C.byref(mid), C.byref(tc)))
        mp = (C.c_int * 16)()
        mma = C.c_int()
        check(lib().svb_plan_phase_map(self._h, p, f, mp, C.byref(mma)))
        return {"R": list(R), "op_begin": b.value, "op_end": e.value, "flags": fl.value,
                "op_mid": mid.value, "tc": tc.value, "map": list(mp), "mma": bool(mma.value)}

    def tc_matrix(self, p: int, tc: int) -> np.ndarray:
        out = np.zeros(2 * 1024, dtype=np.float64)
        n = check(lib().svb_plan_tc_matrix(self._h, p, tc, _dptr(out), 1024))
        d = int(round(n ** 0.5))
        return out[:2 * n].view(np.complex128).reshape(d, d).copy()

    def phase_op(self, p: int, i: int) -> dict:
        kind, k, mask = C.c_int(), C.c_int(), C.c_int()
        src = np.zeros(2 * SVB_MAX_TARGETS, dtype=np.int32)
        co = np.zeros(2 * 4096, dtype=np.float64)
        n = check(lib().svb_plan_phase_op(self._h, p, i, C.byref(kind), C.byref(k), C.byref(mask),
                                          _iptr(src), _dptr(co), 4096))
        out = {"kind": KINDS[kind.value], "k": k.value, "mask": mask.value,
               "coeffs": co[:2 * n].view(np.complex128).copy()}
        if kind.value == 2:  # CNOT: control / target register bits
            out["ctrl"], out["tgt"] = int(src[0]), int(src[1])
        if kind.value == 3:  # controlled op: target register mask; control thread bit, or
            # (negative) the shard qubit -1 - src[0] outside the tile
            out["ctrl_thread_bit"] = int(src[0])
        if kind.value == 1:
            out["thread_bits"] = [int(x) for x in src[:mask.value]]
            out["rmap"] = src[8:16].view(np.uint8).copy()
            kx, xm = C.c_int(), C.c_ulonglong()
            check(lib().svb_plan_phase_op_ext(self._h, p, i, C.byref(kx), C.byref(xm)))
            out["ext_qubits"] = [q for q in range(64) if (xm.value >> q) & 1]
            assert len(out["ext_qubits"]) == kx.value
        return out

    def pass_gates(self, p: int) -> list[int]:
        buf = np.zeros(max(1, self.num_gates), dtype=np.int32)
        n = check(lib().svb_plan_pass_gates(self._h, p, _iptr(buf), int(buf.size)))
        return [int(x) for x in buf[:n]]

    def kernel_op(self, p: int, i: int) -> dict:
        kind, k = C.c_int(), C.c_int()
        tg = np.zeros(SVB_MAX_TARGETS, dtype=np.int32)
        co = np.zeros(2 * 4096, dtype=np.float64)
        n = check(lib().svb_plan_kernel_op(self._h, p, i, C.byref(kind), C.byref(k), _iptr(tg),
                                           _dptr(co), 4096))
        coeffs = co[:2 * n].view(np.complex128).copy()
        out = {"kind": KINDS[kind.value], "k": k.value,
               "targets": [int(t) for t in tg[:k.value]], "coeffs": coeffs}
        if kind.value == 3:  # controlled op: U0 / U1 on targets[0], control = shard qubit outside the tile
            out["ctrl_qubit"] = int(tg[1])
        return out

    def execute(self, amps_ptr: int, stream: int, first: int = 0, count: int | None = None):
        if count is None:
            count = self.num_passes() - first
        check(lib().svb_plan_execute_range(self._h, C.c_void_p(amps_ptr), first, count,
                                           C.c_void_p(stream)))

    def close(self):
        if self._h is not None and _lib is not None:
            _lib.svb_plan_destroy(self._h)
        self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass


def swap_blocks(a_ptr: int, b_ptr: int, nbytes: int, stream: int) -> None:
    """In-place a <-> b of two device ranges in one kernel (svb_swap_blocks)."""
    check(lib().svb_swap_blocks(C.c_void_p(a_ptr), C.c_void_p(b_ptr), int(nbytes), C.c_void_p(stream)))


def enable_peer_access(device: int, peer: int) -> None:
    check(lib().svb_enable_peer_access(int(device), int(peer)))


def ipc_export(ptr: int) -> tuple[bytes, int]:
    """(64-byte CUDA IPC handle of the allocation holding ptr, ptr's offset in it)."""
    h = (C.c_ubyte * 64)()
    off = C.c_longlong()
    check(lib().svb_ipc_export(C.c_void_p(ptr), h, C.byref(off)))
    return bytes(h), int(off.value)


def ipc_import(handle: bytes, offset: int) -> tuple[int, int]:
    """Map a peer process's allocation: (pointer, base to pass to ipc_close)."""
    h = (C.c_ubyte * 64).from_buffer_copy(handle)
    ptr, base = C.c_void_p(), C.c_void_p()
    check(lib().svb_ipc_import(h, int(offset), C.byref(ptr), C.byref(base)))
    return int(ptr.value), int(base.value)


def ipc_close(base: int) -> None:
    check(lib().svb_ipc_close(C.c_void_p(base)))
