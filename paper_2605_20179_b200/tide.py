"""ctypes binding of libtide.so (include/tide.h) -- argument marshalling only.

Every step of the TIDE layer-step runs in the CUDA kernels of libtide.so.  This
module turns torch tensors into device pointers and the current torch stream
into a cudaStream_t; it has no compute of its own and no CPU fallback: if the
shared library is missing or the device is not sm_100, it raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libtide.so")

TIDE_OK, TIDE_EINVAL, TIDE_ECAPACITY, TIDE_EPLACEMENT, TIDE_ECUDA, TIDE_ENCCL, TIDE_ENOMEM, \
    TIDE_EUNSUPPORTED = range(8)
ABI_VERSION = 2  # include/tide.h TIDE_ABI_VERSION
TIDE_F32, TIDE_BF16 = 0, 1
TIDE_NORM_TOPK, TIDE_SHARED_EXPERT, TIDE_LAZY_PROMOTE = 1, 2, 4
TIDE_COUNTER_WINDOW, TIDE_COUNTER_CUMULATIVE, TIDE_TIE_INCUMBENT = 8, 16, 32

STATUS_NAMES = {0: "TIDE_OK", 1: "TIDE_EINVAL", 2: "TIDE_ECAPACITY", 3: "TIDE_EPLACEMENT",
                4: "TIDE_ECUDA", 5: "TIDE_ENCCL", 6: "TIDE_ENOMEM", 7: "TIDE_EUNSUPPORTED"}

EXPORTED = ("tide_abi_version", "tide_build_sm", "tide_last_error", "tide_expert_elems",
            "tide_expert_bytes", "tide_pack_expert", "tide_ctx_create", "tide_ctx_destroy",
            "tide_moe_step", "tide_ctx_set_timing", "tide_ctx_get_timing", "tide_nccl_unique_id",
            "tide_ctx_create_ep", "tide_ctx_create_ep_like", "tide_moe_step_ep",
            "tide_interval_cost", "tide_optimize_interval", "tide_trace_stats",
            "tide_ctx_create_ep_p2p", "tide_ep_handle_bytes", "tide_ctx_ep_export",
            "tide_ctx_ep_connect", "tide_ctx_ep_error", "tide_ctx_ep_wait", "tide_interval_profile",
            "tide_interval_cost_trace", "tide_optimize_interval_trace", "tide_interval_replay",
            "tide_optimize_interval_replay")


class TideError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


class LayerDesc(ctypes.Structure):
    _fields_ = [("num_experts", ctypes.c_int32), ("top_k", ctypes.c_int32),
                ("hidden", ctypes.c_int32), ("ffn", ctypes.c_int32),
                ("max_tokens", ctypes.c_int32), ("dtype", ctypes.c_int32),
                ("flags", ctypes.c_uint32)]


class ExpertWeights(ctypes.Structure):
    _fields_ = [("device_all", ctypes.c_void_p), ("host_master", ctypes.c_void_p),
                ("shared_w", ctypes.c_void_p)]


class StepStats(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "refreshed", "resident_pairs", "nonresident_pairs", "promotions", "evictions",
        "unique_experts", "experts_streamed", "copies")] + [
        ("h2d_bytes", ctypes.c_int64), ("weight_bytes_read", ctypes.c_int64),
        ("resident_weight_bytes", ctypes.c_int64), ("resident_rows", ctypes.c_int32),
        ("ffn_launches", ctypes.c_int32)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class StepDebug(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("topk_idx", "gates", "pos", "order", "offsets",
                                                "logits", "route_trace", "ffn_trace",
                                                "ffn_item_trace")]


class PhaseTimes(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("router_ms", "route_ms", "gather_ms", "ffn_ms",
                                                "staged_ms", "combine_ms", "total_ms")] + [
        ("steps", ctypes.c_int64), ("launches", ctypes.c_int64), ("ffn_launches", ctypes.c_int64)]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class IntervalModel(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("B", ctypes.c_int32), ("d", ctypes.c_double),
                ("c_io", ctypes.c_double), ("c_miss", ctypes.c_double)]


class IntervalTraceModel(ctypes.Structure):
    _fields_ = [("T", ctypes.c_int32), ("c_io", ctypes.c_double), ("c_step", ctypes.c_double),
                ("miss_lag", ctypes.c_void_p), ("mig_lag", ctypes.c_void_p)]


class IntervalReplayModel(ctypes.Structure):
    _fields_ = [("counts", ctypes.c_void_p), ("T", ctypes.c_int32), ("E", ctypes.c_int32),
                ("B", ctypes.c_int32), ("lazy", ctypes.c_int32), ("passes", ctypes.c_int32),
                ("c_io", ctypes.c_double), ("c_step", ctypes.c_double)]


_lib = None


def lib():
    """Load libtide.so; raise loudly if it is missing (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                              "(nvcc, sm_100a); there is no CPU fallback")
        L = ctypes.CDLL(LIB_PATH)
        L.tide_last_error.restype = ctypes.c_char_p
        L.tide_expert_elems.restype = ctypes.c_size_t
        L.tide_expert_bytes.restype = ctypes.c_size_t
        L.tide_expert_elems.argtypes = [ctypes.POINTER(LayerDesc)]
        L.tide_expert_bytes.argtypes = [ctypes.POINTER(LayerDesc)]
        L.tide_ctx_create.argtypes = [ctypes.POINTER(LayerDesc), ctypes.c_int32, ctypes.c_int32,
                                      ctypes.c_int32, ctypes.POINTER(ctypes.c_void_p)]
        L.tide_ctx_destroy.argtypes = [ctypes.c_void_p]
        L.tide_ctx_destroy.restype = None
        L.tide_pack_expert.argtypes = [ctypes.POINTER(LayerDesc)] + [ctypes.c_void_p] * 5
        L.tide_moe_step.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p,
            ctypes.POINTER(ExpertWeights), ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.POINTER(StepStats), ctypes.POINTER(StepDebug), ctypes.c_void_p]
        L.tide_nccl_unique_id.argtypes = [ctypes.c_void_p]
        L.tide_ctx_create_ep.argtypes = [ctypes.POINTER(LayerDesc), ctypes.c_int32, ctypes.c_void_p,
                                         ctypes.c_int32, ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_void_p)]
        L.tide_ctx_create_ep_like.argtypes = [ctypes.POINTER(LayerDesc), ctypes.c_void_p,
                                              ctypes.POINTER(ctypes.c_void_p)]
        L.tide_moe_step_ep.argtypes = [
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32, ctypes.c_int32,
            ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.POINTER(StepStats),
            ctypes.c_void_p]
        L.tide_interval_cost.argtypes = [ctypes.POINTER(IntervalModel), ctypes.c_int32,
                                         ctypes.POINTER(ctypes.c_double),
                                         ctypes.POINTER(ctypes.c_double)]
        L.tide_optimize_interval.argtypes = [ctypes.POINTER(IntervalModel),
                                             ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p]
        L.tide_trace_stats.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                       ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p, ctypes.c_void_p]
        L.tide_ctx_set_timing.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.tide_ctx_set_prefetch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                            ctypes.c_int64]
        L.tide_ctx_get_timing.argtypes = [ctypes.c_void_p, ctypes.POINTER(PhaseTimes)]
        L.tide_ctx_create_ep_p2p.argtypes = [ctypes.POINTER(LayerDesc), ctypes.c_int32,
                                             ctypes.c_int32, ctypes.c_int32,
                                             ctypes.POINTER(ctypes.c_void_p)]
        L.tide_ep_handle_bytes.restype = ctypes.c_size_t
        L.tide_ep_handle_bytes.argtypes = []
        L.tide_ctx_ep_export.argtypes = [ctypes.c_void_p, ctypes.c_void_p,
                                         ctypes.POINTER(ctypes.c_void_p)]
        L.tide_ctx_ep_connect.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        L.tide_ctx_ep_error.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_int32)]
        L.tide_ctx_ep_wait.argtypes = [ctypes.c_void_p, ctypes.c_int32]
        L.tide_interval_profile.argtypes = [ctypes.c_void_p, ctypes.c_int32, ctypes.c_int32,
                                            ctypes.c_int32, ctypes.c_void_p, ctypes.c_void_p]
        L.tide_interval_cost_trace.argtypes = [ctypes.POINTER(IntervalTraceModel), ctypes.c_int32,
                                               ctypes.POINTER(ctypes.c_double),
                                               ctypes.POINTER(ctypes.c_double)]
        L.tide_optimize_interval_trace.argtypes = [ctypes.POINTER(IntervalTraceModel),
                                                   ctypes.POINTER(ctypes.c_int32), ctypes.c_void_p]
        L.tide_interval_replay.argtypes = [ctypes.c_void_p] + [ctypes.c_int32] * 6 + [
            ctypes.POINTER(ctypes.c_int64), ctypes.c_void_p]
        L.tide_optimize_interval_replay.argtypes = [ctypes.POINTER(IntervalReplayModel),
                                                    ctypes.c_int32, ctypes.POINTER(ctypes.c_int32),
                                                    ctypes.c_void_p]
        _lib = L
    return _lib


def _check(status: int):
    if status != TIDE_OK:
        raise TideError(status, lib().tide_last_error().decode(errors="replace"))


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream_ptr(stream=None):
    s = torch.cuda.current_stream() if stream is None else stream
    return ctypes.c_void_p(s.cuda_stream)


def torch_dtype(code: int):
    return torch.bfloat16 if code == TIDE_BF16 else torch.float32


def make_desc(num_experts, top_k, hidden, ffn, max_tokens, dtype=TIDE_BF16,
              norm_topk=True, shared_expert=False, lazy_promote=False, counter="current",
              incumbent_ties=False) -> LayerDesc:
    """counter: "current" (R-5), "window" or "cumulative" (NEXT-1)."""
    flags = (TIDE_NORM_TOPK if norm_topk else 0) | (TIDE_SHARED_EXPERT if shared_expert else 0) \
        | (TIDE_LAZY_PROMOTE if lazy_promote else 0) \
        | {"current": 0, "window": TIDE_COUNTER_WINDOW,
           "cumulative": TIDE_COUNTER_CUMULATIVE}[counter] \
        | (TIDE_TIE_INCUMBENT if incumbent_ties else 0)
    return LayerDesc(num_experts, top_k, hidden, ffn, max_tokens, dtype, flags)


def expert_elems(desc: LayerDesc) -> int:
    return lib().tide_expert_elems(ctypes.byref(desc))


def expert_bytes(desc: LayerDesc) -> int:
    return lib().tide_expert_bytes(ctypes.byref(desc))


def pack_expert(desc: LayerDesc, w_gate, w_up, w_down, dst, stream=None):
    """tide_pack_expert: [Wg; Wu; Wd] -> dst (host or device tensors)."""
    _check(lib().tide_pack_expert(ctypes.byref(desc), _ptr(w_gate), _ptr(w_up), _ptr(w_down),
                                  _ptr(dst), _stream_ptr(stream)))


@dataclass
class StepOutputs:
    out: torch.Tensor
    hit_counts: torch.Tensor
    placement: torch.Tensor
    stats: dict | None
    debug: dict | None


class Context:
    """One tide_ctx (one MoE layer on one device)."""

    def __init__(self, desc: LayerDesc, capacity: int, staging_slots: int = 16, device: int = 0):
        h = ctypes.c_void_p()
        _check(lib().tide_ctx_create(ctypes.byref(desc), capacity, staging_slots, device,
                                     ctypes.byref(h)))
        self.handle = h
        self.desc = desc
        self.capacity = capacity
        self.device = device

    def close(self):
        if self.handle:
            lib().tide_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_timing(self, enable: bool = True):
        """tide_ctx_set_timing: per-phase CUDA-event timing on the step stream."""
        _check(lib().tide_ctx_set_timing(self.handle, int(enable)))

    def timing(self) -> dict:
        t = PhaseTimes()
        _check(lib().tide_ctx_get_timing(self.handle, ctypes.byref(t)))
        return t.as_dict()

    def set_prefetch(self, next_ctx: "Context | None", next_device_all=None,
                     budget_bytes: int = 0):
        """tide_ctx_set_prefetch: prefetch `next_ctx`'s likely experts into L2 at the end of
        this context's FFN (NEXT-3; next_device_all = its packed experts), or, with
        next_device_all None (next serves from a pinned host master), copy its predicted
        streamed experts host-to-HBM into its prefetch slots; None / 0 disables."""
        _check(lib().tide_ctx_set_prefetch(
            self.handle, next_ctx.handle if next_ctx is not None else None,
            _ptr(next_device_all) if next_device_all is not None else None, int(budget_bytes)))

    def moe_step(self, block_hidden, router_w, *, device_all=None, host_master=None,
                 shared_w=None, placement, step: int, interval: int, capacity: int | None = None,
                 out=None, hit_counts=None, placement_out=None, stats: bool = False,
                 debug: bool | str = False, stream=None) -> StepOutputs:
        """tide_moe_step.  Tensors: block_hidden [N,H] (device), router_w [E,H] (device),
        device_all [E, 3HF] device or host_master [E, 3HF] pinned host, shared_w [3HF]
        device, placement [E] uint8 device.  debug: True (routing outputs, logits and kernel
        timestamps), "routing" (top-k, gates, pos, order, offsets only) or "trace"
        (timestamps only); test instrumentation, returned in StepOutputs.debug."""
        d = self.desc
        N = block_hidden.shape[0]
        dev = block_hidden.device
        if out is None:
            out = torch.empty(N, d.hidden, dtype=block_hidden.dtype, device=dev)
        if hit_counts is None:
            hit_counts = torch.empty(d.num_experts, dtype=torch.int32, device=dev)
        if placement_out is None:
            placement_out = torch.empty(d.num_experts, dtype=torch.uint8, device=dev)
        w = ExpertWeights(None if device_all is None else device_all.data_ptr(),
                          None if host_master is None else host_master.data_ptr(),
                          None if shared_w is None else shared_w.data_ptr())
        st = StepStats() if stats else None
        dbg_t = None
        dbg = None
        if debug:
            k, E = d.top_k, d.num_experts
            dbg_t = {"topk_idx": torch.empty(N, k, dtype=torch.int32, device=dev),
                     "gates": torch.empty(N, k, dtype=torch.float32, device=dev),
                     "pos": torch.empty(N, k, dtype=torch.int32, device=dev),
                     "order": torch.empty(E, dtype=torch.int32, device=dev),
                     "offsets": torch.empty(E + 1, dtype=torch.int32, device=dev),
                     "logits": torch.empty(N, E, dtype=torch.float32, device=dev),
                     "route_trace": torch.zeros(4 * ((E + 7) // 8) * max(1, N),
                                                dtype=torch.int64, device=dev),
                     "ffn_trace": torch.zeros(8 * torch.cuda.get_device_properties(dev).multi_processor_count,
                                              dtype=torch.int64, device=dev),
                     "ffn_item_trace": torch.zeros(
                         4 * 64 * torch.cuda.get_device_properties(dev).multi_processor_count,
                         dtype=torch.int64, device=dev)}
            if debug == "trace":  # kernel timestamps only: no extra copies on the stream
                dbg_t = {n: (v if n.endswith("_trace") else None) for n, v in dbg_t.items()}
            elif debug == "routing":  # the routing outputs only (D2D copies, graph-capturable)
                dbg_t = {n: (None if n.endswith("_trace") or n == "logits" else v)
                         for n, v in dbg_t.items()}
            dbg = StepDebug(*((dbg_t[n].data_ptr() if dbg_t[n] is not None else None)
                              for n, _ in StepDebug._fields_))
        _check(lib().tide_moe_step(
            self.handle, _ptr(block_hidden), N, _ptr(router_w), ctypes.byref(w), _ptr(placement),
            step, interval, self.capacity if capacity is None else capacity, _ptr(out),
            _ptr(hit_counts), _ptr(placement_out), ctypes.byref(st) if st is not None else None,
            ctypes.byref(dbg) if dbg is not None else None, _stream_ptr(stream)))
        return StepOutputs(out, hit_counts, placement_out, st.as_dict() if st else None, dbg_t)


def pack_layer(desc: LayerDesc, wg, wu, wd, out=None):
    """Pack E experts ([E,F,H], [E,F,H], [E,H,F] tensors, any device) into
    [E, 3HF] (allocated on wg's device if ``out`` is None)."""
    E = wg.shape[0]
    n = expert_elems(desc)
    if out is None:
        out = torch.empty(E, n, dtype=wg.dtype, device=wg.device)
    for e in range(E):
        pack_expert(desc, wg[e], wu[e], wd[e], out[e])
    return out


def nccl_unique_id() -> bytes:
    """tide_nccl_unique_id: 128 bytes to share with every rank."""
    buf = ctypes.create_string_buffer(128)
    _check(lib().tide_nccl_unique_id(buf))
    return buf.raw


class EPContext(Context):
    """tide_ctx_create_ep: expert-parallel context (rank of world), own NCCL communicator."""

    def __init__(self, desc: LayerDesc, unique_id: bytes | None, rank: int, world: int,
                 device: int = 0, like: "EPContext | None" = None):
        h = ctypes.c_void_p()
        if like is not None:  # share `like`'s NCCL communicator
            _check(lib().tide_ctx_create_ep_like(ctypes.byref(desc), like.handle, ctypes.byref(h)))
        else:
            uid = ctypes.create_string_buffer(bytes(unique_id), 128)
            _check(lib().tide_ctx_create_ep(ctypes.byref(desc), device, uid, rank, world,
                                            ctypes.byref(h)))
        self.handle = h
        self.desc = desc
        self.rank, self.world = rank, world
        self.local_experts = desc.num_experts // world
        self.capacity = self.local_experts
        self.device = device

    def wait(self, timeout_ms: int = 20000):
        """tide_ctx_ep_wait: host wait for the last step with NCCL async-error polling; raises
        TideError (TIDE_ENCCL / TIDE_ECUDA) on a communicator error, a peer-memory wait that
        gave up, or a timeout."""
        _check(lib().tide_ctx_ep_wait(self.handle, int(timeout_ms)))

    def moe_step_ep(self, block_hidden, router_w, local_experts, *, shared_w=None, placement,
                    step: int, interval: int, capacity: int | None = None, out=None,
                    hit_counts=None, placement_out=None, stats: bool = False,
                    stream=None) -> StepOutputs:
        """tide_moe_step_ep: local_experts [E/P, 3HF] device (this rank's experts),
        placement [E/P] uint8 device; hit_counts [E] (global)."""
        d = self.desc
        N = block_hidden.shape[0]
        dev = block_hidden.device
        if out is None:
            out = torch.empty(N, d.hidden, dtype=block_hidden.dtype, device=dev)
        if hit_counts is None:
            hit_counts = torch.empty(d.num_experts, dtype=torch.int32, device=dev)
        if placement_out is None:
            placement_out = torch.empty(self.local_experts, dtype=torch.uint8, device=dev)
        st = StepStats() if stats else None
        _check(lib().tide_moe_step_ep(
            self.handle, _ptr(block_hidden), N, _ptr(router_w), _ptr(local_experts),
            _ptr(shared_w), _ptr(placement), step, interval,
            self.capacity if capacity is None else capacity, _ptr(out), _ptr(hit_counts),
            _ptr(placement_out), ctypes.byref(st) if st is not None else None,
            _stream_ptr(stream)))
        return StepOutputs(out, hit_counts, placement_out, st.as_dict() if st else None, None)


class EPPeerContext(EPContext):
    """tide_ctx_create_ep_p2p: expert-parallel context whose dispatch and combine are done by
    the kernels over peer memory (no NCCL on the data path).  Connect it before stepping:
    `export()` on every rank, exchange, `connect(handles, bases)` on every rank, barrier."""

    def __init__(self, desc: LayerDesc, rank: int, world: int, device: int = 0):
        h = ctypes.c_void_p()
        _check(lib().tide_ctx_create_ep_p2p(ctypes.byref(desc), device, rank, world,
                                            ctypes.byref(h)))
        self.handle = h
        self.desc = desc
        self.rank, self.world = rank, world
        self.local_experts = desc.num_experts // world
        self.capacity = self.local_experts
        self.device = device

    def export(self) -> tuple[bytes, int]:
        """(IPC handle bytes, device base pointer) of this rank's symmetric region."""
        n = lib().tide_ep_handle_bytes()
        buf = ctypes.create_string_buffer(n)
        base = ctypes.c_void_p()
        _check(lib().tide_ctx_ep_export(self.handle, buf, ctypes.byref(base)))
        return buf.raw, int(base.value or 0)

    def connect(self, handles: list[bytes] | None = None, bases: list[int | None] | None = None):
        """handles: every rank's export()[0] in rank order (other processes); bases: every
        rank's export()[1] where the region is directly addressable (same process)."""
        n = lib().tide_ep_handle_bytes()
        hb = None
        if handles is not None:
            hb = ctypes.create_string_buffer(b"".join(bytes(x).ljust(n, b"\0")[:n] for x in handles),
                                             n * self.world)
        bb = None
        if bases is not None:
            bb = (ctypes.c_void_p * self.world)(*[b or None for b in bases])
        _check(lib().tide_ctx_ep_connect(self.handle, hb, bb))

    def error(self) -> int:
        v = ctypes.c_int32()
        _check(lib().tide_ctx_ep_error(self.handle, ctypes.byref(v)))
        return v.value


def interval_cost(T: int, B: int, d: float, c_io: float, c_miss: float, tau: int):
    """tide_interval_cost -> (Eq. 5 I/O cost, Eq. 6 miss cost)."""
    m = IntervalModel(T, B, d, c_io, c_miss)
    io, ms = ctypes.c_double(), ctypes.c_double()
    _check(lib().tide_interval_cost(ctypes.byref(m), tau, ctypes.byref(io), ctypes.byref(ms)))
    return io.value, ms.value


def optimize_interval(T: int, B: int, d: float, c_io: float, c_miss: float):
    """tide_optimize_interval -> (tau*, [total cost for tau = 1..T-1])."""
    import numpy as np
    m = IntervalModel(T, B, d, c_io, c_miss)
    tau = ctypes.c_int32()
    curve = np.zeros(max(1, T - 1), np.float64)
    _check(lib().tide_optimize_interval(ctypes.byref(m), ctypes.byref(tau),
                                        ctypes.c_void_p(curve.ctypes.data)))
    return tau.value, curve


def trace_stats(counts, B: int, stream=None):
    """tide_trace_stats on a device [T, E] int32 tensor -> (sim [T,T] f64, unique [T], drift [T-1])."""
    T, E = counts.shape
    dev = counts.device
    sim = torch.empty(T, T, dtype=torch.float64, device=dev)
    uniq = torch.empty(T, dtype=torch.int32, device=dev)
    drift = torch.empty(max(1, T - 1), dtype=torch.float64, device=dev)
    _check(lib().tide_trace_stats(_ptr(counts.contiguous()), T, E, B, _ptr(sim), _ptr(uniq),
                                  _ptr(drift), _stream_ptr(stream)))
    return sim, uniq, drift[: T - 1]


def interval_profile(counts, B: int):
    """tide_interval_profile on a host [T, E] int32 array -> (miss_lag [T], mig_lag [T])."""
    import numpy as np
    c = np.ascontiguousarray(counts, np.int32)
    T, E = c.shape
    miss = np.zeros(T, np.float64)
    mig = np.zeros(T, np.float64)
    _check(lib().tide_interval_profile(ctypes.c_void_p(c.ctypes.data), T, E, B,
                                       ctypes.c_void_p(miss.ctypes.data),
                                       ctypes.c_void_p(mig.ctypes.data)))
    return miss, mig


def _trace_model(T, c_io, c_step, miss_lag, mig_lag):
    import numpy as np
    miss = np.ascontiguousarray(miss_lag, np.float64)
    mig = np.ascontiguousarray(mig_lag, np.float64)
    m = IntervalTraceModel(T, c_io, c_step, ctypes.c_void_p(miss.ctypes.data),
                           ctypes.c_void_p(mig.ctypes.data))
    return m, (miss, mig)


def interval_cost_trace(T, c_io, c_step, miss_lag, mig_lag, tau):
    """tide_interval_cost_trace -> (expert copies over the block, cost)."""
    m, keep = _trace_model(T, c_io, c_step, miss_lag, mig_lag)
    cp, c = ctypes.c_double(), ctypes.c_double()
    _check(lib().tide_interval_cost_trace(ctypes.byref(m), tau, ctypes.byref(cp), ctypes.byref(c)))
    return cp.value, c.value


def optimize_interval_trace(T, c_io, c_step, miss_lag, mig_lag):
    """tide_optimize_interval_trace -> (tau*, [cost for tau = 1..T-1])."""
    import numpy as np
    m, keep = _trace_model(T, c_io, c_step, miss_lag, mig_lag)
    tau = ctypes.c_int32()
    curve = np.zeros(max(1, T - 1), np.float64)
    _check(lib().tide_optimize_interval_trace(ctypes.byref(m), ctypes.byref(tau),
                                              ctypes.c_void_p(curve.ctypes.data)))
    return tau.value, curve


def interval_replay(counts, B: int, tau: int, lazy: bool = False, passes: int = 2):
    """tide_interval_replay on a host [T, E] int32 trace -> (copies of the last pass, [T])."""
    import numpy as np
    c = np.ascontiguousarray(counts, np.int32)
    T, E = c.shape
    per = np.zeros(T, np.int32)
    cp = ctypes.c_int64()
    _check(lib().tide_interval_replay(ctypes.c_void_p(c.ctypes.data), T, E, B, tau, int(lazy),
                                      passes, ctypes.byref(cp), ctypes.c_void_p(per.ctypes.data)))
    return cp.value, per


def optimize_interval_replay(counts, B: int, c_io: float, c_step: float, tau_max: int,
                             lazy: bool = False, passes: int = 2):
    """tide_optimize_interval_replay -> (tau*, [cost for tau = 1..tau_max])."""
    import numpy as np
    c = np.ascontiguousarray(counts, np.int32)
    T, E = c.shape
    m = IntervalReplayModel(ctypes.c_void_p(c.ctypes.data), T, E, B, int(lazy), passes, c_io, c_step)
    tau = ctypes.c_int32()
    curve = np.zeros(tau_max, np.float64)
    _check(lib().tide_optimize_interval_replay(ctypes.byref(m), tau_max, ctypes.byref(tau),
                                               ctypes.c_void_p(curve.ctypes.data)))
    return tau.value, curve
