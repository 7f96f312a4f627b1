"""Seeded synthetic inputs for the TIDE MoE layer-step (shared by tests, bench
and oracle callers).  Holds NO arithmetic of the method: only random numbers,
shapes and dtype conversions.  Recipe: DESIGN.md "Input recipe".

Weights come from a counter-based hash (murmur3 fmix32 over a Weyl sequence),
so any expert of any layer can be generated independently, on the host
(NumPy) or on the device (torch int64 ops) with identical bits.  Activations
come from NumPy's PCG64 (host) or torch's Philox (device); they are passed to
both sides as stored bytes, so they need not match across implementations.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

M32 = 0xFFFFFFFF
_C1, _C2, _GOLD = 0x85EBCA6B, 0xC2B2AE35, 0x9E3779B1


# ----------------------------------------------------------------- configs
@dataclass(frozen=True)
class Shape:
    """One row of BASELINE.json configs."""
    name: str
    num_experts: int
    top_k: int
    hidden: int
    ffn: int
    layers: int
    tokens: int          # tokens per layer-step (block length x blocks)
    steps: int = 32      # denoising steps per block (DESIGN R-19)
    interval: int = 2
    capacity: int | None = None
    dtype: str = "bf16"  # weights and activations
    shared_expert: bool = False
    extra: dict = field(default_factory=dict, hash=False, compare=False)

    @property
    def expert_bytes(self) -> int:
        return 3 * self.hidden * self.ffn * (2 if self.dtype == "bf16" else 4)


TOY = Shape("toy", 16, 2, 64, 128, 1, 8, steps=8, interval=2, capacity=4, dtype="f32")
MINI = Shape("mini", 256, 8, 2048, 512, 20, 32, shared_expert=True)
FLASH = Shape("flash", 256, 8, 4096, 1024, 32, 32)
SWEEP = Shape("sweep", 256, 8, 2048, 512, 20, 256, shared_expert=True)
SHAPES = {s.name: s for s in (TOY, MINI, FLASH, SWEEP)}

# calibrated temporal-routing constants (the statistics they reproduce are pinned
# in tests/test_next_rows.py::test_generator_matches_paper_routing_statistics)
ALPHA, SKEW, A0 = 0.99, 0.5, 0.8


# ------------------------------------------------------------- bf16 helpers
def f32_to_bf16_bits(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even fp32 -> bf16, returned as uint16 bit patterns."""
    b = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    r = (b + 0x7FFF + ((b >> 16) & 1)) >> 16
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.ascontiguousarray(b, np.uint16).astype(np.uint32) << 16).view(np.float32)


# ------------------------------------------------------------ counter hash
def _key(seed: int, *tags: int) -> int:
    """Host-side 32-bit key for (seed, tags...) -- splitmix64 chain."""
    z = seed & 0xFFFFFFFFFFFFFFFF
    for t in (0x5EED,) + tuple(tags):
        z = (z + 0x9E3779B97F4A7C15 + (t & 0xFFFFFFFFFFFFFFFF)) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & 0xFFFFFFFFFFFFFFFF
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & 0xFFFFFFFFFFFFFFFF
        z ^= z >> 31
    return z & M32


def _fmix_np(h: np.ndarray) -> np.ndarray:
    h = h ^ (h >> 16)
    h = (h * _C1) & M32
    h = h ^ (h >> 13)
    h = (h * _C2) & M32
    return h ^ (h >> 16)


def hash_u32_np(key: int, idx: np.ndarray) -> np.ndarray:
    h = ((idx.astype(np.int64) * _GOLD + key) & M32).astype(np.int64)
    return _fmix_np(h)


def uniform_np(key: int, n: int, bound: float) -> np.ndarray:
    """n fp32 values uniform in [-bound, bound): (2u-1)*bound, u = (h>>8)/2^24."""
    h = hash_u32_np(key, np.arange(n, dtype=np.int64))
    u = (h >> 8).astype(np.float32) * np.float32(2.0 ** -24)
    t = u * np.float32(2.0) - np.float32(1.0)
    return t * np.float32(bound)


def _store(a32: np.ndarray, dtype: str) -> np.ndarray:
    return f32_to_bf16_bits(a32) if dtype == "bf16" else a32.astype(np.float32)


# tensor tags
T_WR, T_WG, T_WU, T_WD, T_SG, T_SU, T_SD, T_PERM = range(1, 9)


def expert_np(shape: Shape, seed: int, layer: int, e: int):
    """(wg [F,H], wu [F,H], wd [H,F]) of routed expert e, stored dtype."""
    H, F = shape.hidden, shape.ffn
    wg = uniform_np(_key(seed, layer, T_WG, e), F * H, math.sqrt(3.0 / H)).reshape(F, H)
    wu = uniform_np(_key(seed, layer, T_WU, e), F * H, math.sqrt(3.0 / H)).reshape(F, H)
    wd = uniform_np(_key(seed, layer, T_WD, e), H * F, math.sqrt(3.0 / F)).reshape(H, F)
    return tuple(_store(a, shape.dtype) for a in (wg, wu, wd))


def shared_np(shape: Shape, seed: int, layer: int):
    H, F = shape.hidden, shape.ffn
    wg = uniform_np(_key(seed, layer, T_SG), F * H, math.sqrt(3.0 / H)).reshape(F, H)
    wu = uniform_np(_key(seed, layer, T_SU), F * H, math.sqrt(3.0 / H)).reshape(F, H)
    wd = uniform_np(_key(seed, layer, T_SD), H * F, math.sqrt(3.0 / F)).reshape(H, F)
    return tuple(_store(a, shape.dtype) for a in (wg, wu, wd))


def popularity_perm(shape: Shape, seed: int, layer: int) -> np.ndarray:
    return np.random.Generator(np.random.PCG64(_key(seed, layer, T_PERM))).permutation(
        shape.num_experts)


def router_np(shape: Shape, seed: int, layer: int, skew: float = SKEW) -> np.ndarray:
    """Wr [E,H] ~ U(+-sqrt(3/H)); column 0 carries the popularity bias
    -skew*ln(1+pi(e)) (x[:,0] == 1), giving skewed expert demand."""
    E, H = shape.num_experts, shape.hidden
    w = uniform_np(_key(seed, layer, T_WR), E * H, math.sqrt(3.0 / H)).reshape(E, H)
    if skew:
        pi = popularity_perm(shape, seed, layer)
        w[:, 0] = (-skew * np.log1p(pi.astype(np.float64))).astype(np.float32)
    return _store(w, shape.dtype)


@dataclass
class LayerTensors:
    wr: np.ndarray
    wg: np.ndarray  # [E,F,H]
    wu: np.ndarray  # [E,F,H]
    wd: np.ndarray  # [E,H,F]
    shared: tuple | None


def layer_np(shape: Shape, seed: int, layer: int = 0, skew: float = SKEW) -> LayerTensors:
    ex = [expert_np(shape, seed, layer, e) for e in range(shape.num_experts)]
    return LayerTensors(router_np(shape, seed, layer, skew),
                        np.stack([t[0] for t in ex]), np.stack([t[1] for t in ex]),
                        np.stack([t[2] for t in ex]),
                        shared_np(shape, seed, layer) if shape.shared_expert else None)


# ----------------------------------------------------------- activations
def block_hidden_np(shape: Shape, seed: int, layer: int = 0, steps: int | None = None,
                    tokens: int | None = None, alpha: float = ALPHA, a0: float = A0,
                    iid: bool = False) -> np.ndarray:
    """[T, N, H] block hidden states (stored dtype), temporal model of
    DESIGN.md: x_t = a_t*mu + sqrt(1-a_t^2)*s_t, s_t = alpha*s_{t-1} +
    sqrt(1-alpha^2)*z_t, a_t = a0*(1-t/T); x[:,0] = 1 (bias column).
    ``iid=True`` gives the uniform stress case (alpha=0, a0=0)."""
    T = shape.steps if steps is None else steps
    N = shape.tokens if tokens is None else tokens
    H = shape.hidden
    if iid:
        alpha, a0 = 0.0, 0.0
    g = np.random.Generator(np.random.PCG64(_key(seed, layer, 0xB10C)))
    mu = g.standard_normal(H)
    s = g.standard_normal((N, H))
    out = np.empty((T, N, H), np.float32)
    for t in range(T):
        if t > 0:
            s = alpha * s + math.sqrt(1 - alpha * alpha) * g.standard_normal((N, H))
        a = a0 * (1 - t / T)
        x = a * mu + math.sqrt(1 - a * a) * s
        x[:, 0] = 1.0
        out[t] = x
    return _store(out, shape.dtype)


def random_placement(E: int, count: int, seed: int) -> np.ndarray:
    g = np.random.Generator(np.random.PCG64(_key(seed, 0x9A7)))
    p = np.zeros(E, np.uint8)
    p[g.choice(E, size=count, replace=False)] = 1
    return p


# ------------------------------------------------- device-side generation
def _fmix_t(h):
    h = h ^ (h >> 16)
    h = (h * _C1) & M32
    h = h ^ (h >> 13)
    h = (h * _C2) & M32
    return h ^ (h >> 16)


def uniform_torch(key: int, n: int, bound: float, device, out_dtype=None):
    """Bit-identical device twin of uniform_np (int64 arithmetic, fp32 ops)."""
    import torch
    idx = torch.arange(n, dtype=torch.int64, device=device)
    h = _fmix_t((idx * _GOLD + key) & M32)
    u = (h >> 8).to(torch.float32) * torch.tensor(2.0 ** -24, dtype=torch.float32, device=device)
    t = u * torch.tensor(2.0, dtype=torch.float32, device=device) - torch.tensor(
        1.0, dtype=torch.float32, device=device)
    v = t * torch.tensor(bound, dtype=torch.float32, device=device)
    return v if out_dtype is None else v.to(out_dtype)


def expert_torch(shape: Shape, seed: int, layer: int, e: int, device):
    import torch
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    H, F = shape.hidden, shape.ffn
    wg = uniform_torch(_key(seed, layer, T_WG, e), F * H, math.sqrt(3.0 / H), device, dt)
    wu = uniform_torch(_key(seed, layer, T_WU, e), F * H, math.sqrt(3.0 / H), device, dt)
    wd = uniform_torch(_key(seed, layer, T_WD, e), H * F, math.sqrt(3.0 / F), device, dt)
    return wg.view(F, H), wu.view(F, H), wd.view(H, F)


def shared_torch(shape: Shape, seed: int, layer: int, device):
    import torch
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    H, F = shape.hidden, shape.ffn
    wg = uniform_torch(_key(seed, layer, T_SG), F * H, math.sqrt(3.0 / H), device, dt)
    wu = uniform_torch(_key(seed, layer, T_SU), F * H, math.sqrt(3.0 / H), device, dt)
    wd = uniform_torch(_key(seed, layer, T_SD), H * F, math.sqrt(3.0 / F), device, dt)
    return wg.view(F, H), wu.view(F, H), wd.view(H, F)


def router_torch(shape: Shape, seed: int, layer: int, device, skew: float = SKEW):
    import torch
    return np_to_torch(router_np(shape, seed, layer, skew), device)


def np_to_torch(a: np.ndarray, device="cpu"):
    """Stored-bytes NumPy array (float32, or uint16 bf16 bits) -> torch tensor."""
    import torch
    a = np.ascontiguousarray(a)
    if a.dtype == np.uint16:
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16).to(device)
    return torch.from_numpy(a.copy()).to(device)


def torch_to_np(t) -> np.ndarray:
    """torch tensor -> stored-bytes NumPy array (bf16 -> uint16 bits)."""
    import torch
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view(np.uint16)
    return t.numpy()


def block_hidden_torch(shape: Shape, seed: int, layer: int, device, steps: int | None = None,
                       tokens: int | None = None, alpha: float = ALPHA, a0: float = A0,
                       iid: bool = False):
    """Device twin of block_hidden_np (same recipe, torch Philox RNG)."""
    import torch
    T = shape.steps if steps is None else steps
    N = shape.tokens if tokens is None else tokens
    H = shape.hidden
    if iid:
        alpha, a0 = 0.0, 0.0
    g = torch.Generator(device=device)
    g.manual_seed(_key(seed, layer, 0xB10C))
    mu = torch.randn(H, generator=g, device=device)
    s = torch.randn(N, H, generator=g, device=device)
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    out = torch.empty(T, N, H, dtype=dt, device=device)
    for t in range(T):
        if t > 0:
            s = alpha * s + math.sqrt(1 - alpha * alpha) * torch.randn(N, H, generator=g,
                                                                      device=device)
        a = a0 * (1 - t / T)
        x = a * mu + math.sqrt(1 - a * a) * s
        x[:, 0] = 1.0
        out[t] = x.to(dt)
    return out


def _uniform_torch_keys(keys, n: int, bound: float, device, out_dtype):
    """Row e of the result == uniform_torch(keys[e], n, bound): one hash stream per key."""
    import torch
    kt = torch.tensor(keys, dtype=torch.int64, device=device)[:, None]
    idx = torch.arange(n, dtype=torch.int64, device=device)[None, :]
    h = _fmix_t((idx * _GOLD + kt) & M32)
    f32 = lambda v: torch.tensor(v, dtype=torch.float32, device=device)  # noqa: E731
    u = (h >> 8).to(torch.float32) * f32(2.0 ** -24)
    return ((u * f32(2.0) - f32(1.0)) * f32(bound)).to(out_dtype)


def layer_torch(shape: Shape, seed: int, layer: int, device, chunk: int = 32,
                skew: float = SKEW, experts: range | None = None):
    """Device twin of layer_np: (wr [E,H], wg [E,F,H], wu [E,F,H], wd [E,H,F], shared|None),
    bit-identical to the host generator, generated `chunk` experts at a time.  `experts`
    (a contiguous id range, e.g. one EP rank's) restricts wg/wu/wd to those experts."""
    import torch
    dt = torch.bfloat16 if shape.dtype == "bf16" else torch.float32
    E, H, F = shape.num_experts, shape.hidden, shape.ffn
    ids = range(E) if experts is None else experts
    n_e = len(ids)
    wg = torch.empty(n_e, F, H, dtype=dt, device=device)
    wu = torch.empty(n_e, F, H, dtype=dt, device=device)
    wd = torch.empty(n_e, H, F, dtype=dt, device=device)
    for i0 in range(0, n_e, chunk):
        es = ids[i0:i0 + chunk]
        for out, tag, n, fan in ((wg, T_WG, F * H, H), (wu, T_WU, F * H, H), (wd, T_WD, H * F, F)):
            keys = [_key(seed, layer, tag, e) for e in es]
            out[i0:i0 + len(es)] = _uniform_torch_keys(keys, n, math.sqrt(3.0 / fan), device,
                                                       dt).view(len(es), *out.shape[1:])
    shared = shared_torch(shape, seed, layer, device) if shape.shared_expert else None
    return router_torch(shape, seed, layer, device, skew=skew), wg, wu, wd, shared
