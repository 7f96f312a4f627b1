"""CPU oracle for the TIDE MoE layer-step (ctypes wrapper over liboracle.so).

TEST INFRASTRUCTURE.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package.  The product path (``paper_2605_20179_b200``) never imports it; it
shares no code with the CUDA path.  Every function here marshals NumPy arrays
into the plain-C fp64 implementation in ``oracle/tide_oracle.c``, whose
functions cite the PAPER.md passages they follow.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "tide_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

F32, BF16 = 0, 1


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (plain C99, fp64, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(
            ["gcc", "-std=c99", "-O2", "-ffp-contract=off", "-fopenmp", "-fPIC", "-shared",
             "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB)
    return _lib


def set_threads(n: int) -> None:
    """Host threads for the oracle's per-token loops (bit-identical results for any n)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None else None


def _dtype_code(a: np.ndarray) -> int:
    if a.dtype == np.float32:
        return F32
    if a.dtype == np.uint16:  # bf16 bit patterns
        return BF16
    raise TypeError(f"oracle inputs are float32 or bf16 bits (uint16), got {a.dtype}")


class _Layer(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "num_experts", "top_k", "hidden", "ffn", "act_dtype", "weight_dtype",
        "router_dtype", "norm_topk", "shared_expert")]


class _IO(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "promotions", "evictions", "experts_streamed", "copies", "resident_pairs",
        "nonresident_pairs")]


def router_logits(x: np.ndarray, wr: np.ndarray) -> np.ndarray:
    N, H = x.shape
    E = wr.shape[0]
    x, wr = np.ascontiguousarray(x), np.ascontiguousarray(wr)
    out = np.empty((N, E), np.float64)
    assert lib().orc_router_logits(N, E, H, _p(x), _dtype_code(x), _p(wr), _dtype_code(wr),
                                   _p(out)) == 0
    return out


def topk(logits: np.ndarray, k: int) -> np.ndarray:
    logits = np.ascontiguousarray(logits, np.float64)
    N, E = logits.shape
    out = np.empty((N, k), np.int32)
    assert lib().orc_topk(N, E, k, _p(logits), _p(out)) == 0
    return out


def gates(logits: np.ndarray, topk_idx: np.ndarray, norm_topk: bool = True) -> np.ndarray:
    logits = np.ascontiguousarray(logits, np.float64)
    topk_idx = np.ascontiguousarray(topk_idx, np.int32)
    N, E = logits.shape
    k = topk_idx.shape[1]
    out = np.empty((N, k), np.float64)
    lib().orc_gates(N, E, k, _p(logits), _p(topk_idx), int(norm_topk), _p(out))
    return out


def hits(topk_idx: np.ndarray, E: int) -> np.ndarray:
    topk_idx = np.ascontiguousarray(topk_idx, np.int32)
    N, k = topk_idx.shape
    out = np.empty(E, np.int32)
    assert lib().orc_hits(N, E, k, _p(topk_idx), _p(out)) == 0
    return out


def is_refresh(step: int, interval: int) -> bool:
    return bool(lib().orc_is_refresh(step, interval))


def placement(hits_: np.ndarray, capacity: int, refresh: bool,
              placement_in: np.ndarray | None = None) -> np.ndarray:
    hits_ = np.ascontiguousarray(hits_, np.int32)
    E = hits_.shape[0]
    pin = np.zeros(E, np.uint8) if placement_in is None else np.ascontiguousarray(placement_in, np.uint8)
    out = np.empty(E, np.uint8)
    assert lib().orc_placement(E, capacity, _p(hits_), int(refresh), _p(pin), _p(out)) == 0
    return out


def buckets(topk_idx: np.ndarray, placement_: np.ndarray):
    topk_idx = np.ascontiguousarray(topk_idx, np.int32)
    placement_ = np.ascontiguousarray(placement_, np.uint8)
    N, k = topk_idx.shape
    E = placement_.shape[0]
    order = np.empty(E, np.int32)
    offsets = np.empty(E + 1, np.int32)
    pos = np.empty((N, k), np.int32)
    lib().orc_buckets(N, E, k, _p(topk_idx), _p(placement_), _p(order), _p(offsets), _p(pos))
    return order, offsets, pos


def swiglu(x: np.ndarray, wg: np.ndarray, wu: np.ndarray, wd: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, np.float64)
    F, H = wg.shape
    wg, wu, wd = (np.ascontiguousarray(a) for a in (wg, wu, wd))
    y = np.empty(H, np.float64)
    lib().orc_swiglu(H, F, _p(x), _p(wg), _p(wu), _p(wd), _dtype_code(wg), _p(y))
    return y


@dataclass
class Layer:
    """One MoE layer's tensors as stored bytes (float32 or bf16 bits as uint16).

    wg, wu: [E, F, H]; wd: [E, H, F]; wr: [E, H]; shared (optional): (wg, wu, wd)
    of one expert.  Any per-expert indexable sequence works (lists of arrays too).
    """
    wr: np.ndarray
    wg: object
    wu: object
    wd: object
    shared: tuple | None = None
    norm_topk: bool = True

    @property
    def E(self):
        return self.wr.shape[0]


def _layer_struct(L: Layer, x: np.ndarray, k: int) -> _Layer:
    wg0 = np.asarray(L.wg[0])
    F, H = wg0.shape
    return _Layer(L.E, k, H, F, _dtype_code(x), _dtype_code(wg0), _dtype_code(L.wr),
                  int(L.norm_topk), int(L.shared is not None))


def _ptr_array(mats, keep):
    arr = (ctypes.c_void_p * len(mats))()
    for i, m in enumerate(mats):
        m = np.ascontiguousarray(m)
        keep.append(m)
        arr[i] = m.ctypes.data
    return arr


@dataclass
class StepResult:
    logits: np.ndarray
    topk_idx: np.ndarray
    gates: np.ndarray
    hits: np.ndarray
    placement: np.ndarray
    order: np.ndarray
    offsets: np.ndarray
    pos: np.ndarray
    out: np.ndarray
    status: int


def moe_step(L: Layer, x: np.ndarray, k: int, placement_in: np.ndarray, step: int,
             interval: int, capacity: int, token_mask: np.ndarray | None = None) -> StepResult:
    x = np.ascontiguousarray(x)
    N, H = x.shape
    E = L.E
    keep: list = []
    st = _layer_struct(L, x, k)
    wg = _ptr_array([L.wg[e] for e in range(E)], keep)
    wu = _ptr_array([L.wu[e] for e in range(E)], keep)
    wd = _ptr_array([L.wd[e] for e in range(E)], keep)
    sh = [np.ascontiguousarray(a) for a in L.shared] if L.shared is not None else [None] * 3
    wr = np.ascontiguousarray(L.wr)
    pin = np.ascontiguousarray(placement_in, np.uint8)
    mask = None if token_mask is None else np.ascontiguousarray(token_mask, np.uint8)
    r = StepResult(np.empty((N, E)), np.empty((N, k), np.int32), np.empty((N, k)),
                   np.empty(E, np.int32), np.empty(E, np.uint8), np.empty(E, np.int32),
                   np.empty(E + 1, np.int32), np.empty((N, k), np.int32), np.empty((N, H)), 0)
    r.status = lib().orc_moe_step(
        ctypes.byref(st), N, _p(x), _p(wr), wg, wu, wd, _p(sh[0]), _p(sh[1]), _p(sh[2]),
        _p(pin), step, interval, capacity, _p(mask), _p(r.logits), _p(r.topk_idx),
        _p(r.gates), _p(r.hits), _p(r.placement), _p(r.order), _p(r.offsets), _p(r.pos),
        _p(r.out))
    return r


def combine(L: Layer, x: np.ndarray, topk_idx: np.ndarray, gates_: np.ndarray,
            token_mask: np.ndarray | None = None) -> np.ndarray:
    """O9 with routing supplied by the caller (used to feed flagged near-tie
    routing from the GPU into the oracle's downstream stages)."""
    x = np.ascontiguousarray(x)
    N, H = x.shape
    k = topk_idx.shape[1]
    keep: list = []
    st = _layer_struct(L, x, k)
    E = L.E
    wg = _ptr_array([L.wg[e] for e in range(E)], keep)
    wu = _ptr_array([L.wu[e] for e in range(E)], keep)
    wd = _ptr_array([L.wd[e] for e in range(E)], keep)
    sh = [np.ascontiguousarray(a) for a in L.shared] if L.shared is not None else [None] * 3
    t = np.ascontiguousarray(topk_idx, np.int32)
    g = np.ascontiguousarray(gates_, np.float64)
    mask = None if token_mask is None else np.ascontiguousarray(token_mask, np.uint8)
    out = np.empty((N, H))
    lib().orc_combine(ctypes.byref(st), N, _p(x), _p(t), _p(g), wg, wu, wd, _p(sh[0]),
                      _p(sh[1]), _p(sh[2]), _p(mask), _p(out))
    return out


def io_step(hits_: np.ndarray, placement_in: np.ndarray, placement_out: np.ndarray,
            loaded: np.ndarray, lazy: bool = False) -> dict:
    """O10.  ``loaded`` (uint8 [E]) is updated in place."""
    assert loaded.dtype == np.uint8 and loaded.flags.c_contiguous
    io = _IO()
    h = np.ascontiguousarray(hits_, np.int32)
    pi = np.ascontiguousarray(placement_in, np.uint8)
    po = np.ascontiguousarray(placement_out, np.uint8)
    lib().orc_io_step(h.shape[0], int(lazy), _p(h), _p(pi), _p(po), _p(loaded), ctypes.byref(io))
    return {n: getattr(io, n) for n, _ in _IO._fields_}


def ep_step(L: Layer, P: int, x: np.ndarray, k: int, placement_in: np.ndarray, step: int,
            interval: int, capacity_per_rank: int):
    x = np.ascontiguousarray(x)
    N, H = x.shape
    E = L.E
    keep: list = []
    st = _layer_struct(L, x, k)
    wg = _ptr_array([L.wg[e] for e in range(E)], keep)
    wu = _ptr_array([L.wu[e] for e in range(E)], keep)
    wd = _ptr_array([L.wd[e] for e in range(E)], keep)
    sh = [np.ascontiguousarray(a) for a in L.shared] if L.shared is not None else [None] * 3
    wr = np.ascontiguousarray(L.wr)
    pin = np.ascontiguousarray(placement_in, np.uint8)
    topk_idx = np.empty((N, k), np.int32)
    h = np.empty(E, np.int32)
    pout = np.empty(E, np.uint8)
    out = np.empty((N, H))
    rc = lib().orc_ep_step(ctypes.byref(st), P, N, _p(x), _p(wr), wg, wu, wd, _p(sh[0]),
                           _p(sh[1]), _p(sh[2]), _p(pin), step,
                           interval, capacity_per_rank, _p(topk_idx), _p(h), _p(pout), _p(out))
    assert rc == 0
    return topk_idx, h, pout, out


# ---------------------------------------------------------------- NEXT-2 / NEXT-4
def _d(fn):
    f = getattr(lib(), fn)
    f.restype = ctypes.c_double
    return f


def migration_cost(tau, B, T, d, c_io=1.0):
    f = _d("orc_migration_cost")
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double]
    return f(tau, B, T, d, c_io)


def miss_fraction(tau, d):
    f = _d("orc_miss_fraction")
    f.argtypes = [ctypes.c_int, ctypes.c_double]
    return f(tau, d)


def miss_cost(tau, B, T, d, c_miss=1.0):
    f = _d("orc_miss_cost")
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double]
    return f(tau, B, T, d, c_miss)


def optimize_tau(T, B, d, c_io, c_miss):
    curve = np.zeros(max(1, T - 1), np.float64)
    f = lib().orc_optimize_tau
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                  ctypes.c_void_p]
    tau = f(T, B, d, c_io, c_miss, _p(curve))
    return tau, curve


def cosine(a, b):
    a = np.ascontiguousarray(a, np.int32)
    b = np.ascontiguousarray(b, np.int32)
    f = _d("orc_cosine")
    f.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return f(a.shape[0], _p(a), _p(b))


def unique(hits_):
    h = np.ascontiguousarray(hits_, np.int32)
    return lib().orc_unique(h.shape[0], _p(h))


def drift(prev, cur, B):
    a = np.ascontiguousarray(prev, np.int32)
    b = np.ascontiguousarray(cur, np.int32)
    f = _d("orc_drift")
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    return f(a.shape[0], B, _p(a), _p(b))


# ---------------------------------------------------------------- NEXT-1
COUNTER_CURRENT, COUNTER_WINDOW, COUNTER_CUMULATIVE = 0, 1, 2


def counter_key(mode, step, hits_, acc):
    h = np.ascontiguousarray(hits_, np.int32)
    a = np.ascontiguousarray(acc, np.int32)
    out = np.empty_like(h)
    lib().orc_counter_key(h.shape[0], mode, step, _p(h), _p(a), _p(out))
    return out


def counter_update(mode, step, refresh, hits_, acc):
    """Updates ``acc`` (int32, contiguous) in place."""
    h = np.ascontiguousarray(hits_, np.int32)
    assert acc.dtype == np.int32 and acc.flags.c_contiguous
    lib().orc_counter_update(h.shape[0], mode, step, int(refresh), _p(h), _p(acc))


def placement_ex(key, capacity, refresh, incumbent_ties, placement_in):
    k_ = np.ascontiguousarray(key, np.int32)
    pin = np.ascontiguousarray(placement_in, np.uint8)
    out = np.empty(k_.shape[0], np.uint8)
    assert lib().orc_placement_ex(k_.shape[0], capacity, _p(k_), int(refresh), int(incumbent_ties),
                                  _p(pin), _p(out)) == 0
    return out


def interval_profile(counts, B):
    """NEXT-2 on B200: (miss_lag [T], mig_lag [T]) of a [T, E] hit-count trace."""
    c = np.ascontiguousarray(counts, np.int32)
    T, E = c.shape
    miss = np.empty(T, np.float64)
    mig = np.empty(T, np.float64)
    assert lib().orc_interval_profile(T, E, B, _p(c), _p(miss), _p(mig)) == 0
    return miss, mig


def interval_replay(counts, B, tau, lazy=False, passes=2):
    """NEXT-2 replay (R-24): (copies of the last pass, copies per step [T]) of a [T, E] trace."""
    c = np.ascontiguousarray(counts, np.int32)
    T, E = c.shape
    per = np.zeros(T, np.int32)
    f = _d("orc_interval_replay")
    f.restype = ctypes.c_long
    f.argtypes = [ctypes.c_int] * 6 + [ctypes.c_void_p, ctypes.c_void_p]
    tot = f(T, E, B, tau, int(lazy), passes, _p(c), _p(per))
    assert tot >= 0
    return int(tot), per


def interval_copies_trace(T, tau, miss_lag, mig_lag):
    f = _d("orc_interval_copies_trace")
    f.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p]
    a = np.ascontiguousarray(miss_lag, np.float64)
    b = np.ascontiguousarray(mig_lag, np.float64)
    return f(T, tau, _p(a), _p(b))
