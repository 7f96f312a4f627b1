"""Shared helpers for the GPU parity tests (test infrastructure: may use oracle/)."""
from __future__ import annotations

import numpy as np
import torch

import oracle
import tidegen as g

TIE_GAP = 1e-6   # BASELINE north_star: logit gaps below 1e-6 are flagged (R-17)
OUT_TOL = 2e-2   # BASELINE north_star: max relative error (R-15)


def desc_for(shape: g.Shape, max_tokens=None, norm_topk=True, lazy=False):
    from paper_2605_20179_b200 import tide
    return tide.make_desc(shape.num_experts, shape.top_k, shape.hidden, shape.ffn,
                          max_tokens or shape.tokens,
                          tide.TIDE_BF16 if shape.dtype == "bf16" else tide.TIDE_F32,
                          norm_topk=norm_topk, shared_expert=shape.shared_expert,
                          lazy_promote=lazy)


class DeviceLayer:
    """One layer's weights on the device (packed) and as host NumPy bytes."""

    def __init__(self, shape: g.Shape, seed: int, layer: int = 0, host_master=False,
                 skew: float = g.SKEW):
        self.shape = shape
        self.np = g.layer_np(shape, seed, layer, skew=skew)
        E = shape.num_experts
        to = lambda a: g.np_to_torch(a)  # noqa: E731
        packed = torch.cat([to(self.np.wg).reshape(E, -1), to(self.np.wu).reshape(E, -1),
                            to(self.np.wd).reshape(E, -1)], dim=1).contiguous()
        self.router = to(self.np.wr).cuda()
        self.device_all = packed.cuda()
        self.host_master = packed.pin_memory() if host_master else None
        self.shared = None
        if self.np.shared is not None:
            self.shared = torch.cat([to(a).reshape(-1) for a in self.np.shared]).cuda()

    def oracle_layer(self, norm_topk=True) -> oracle.Layer:
        n = self.np
        return oracle.Layer(n.wr, n.wg, n.wu, n.wd, n.shared, norm_topk=norm_topk)

    def weights(self, mode="device_all"):
        if mode == "device_all":
            return dict(device_all=self.device_all, shared_w=self.shared)
        return dict(host_master=self.host_master, shared_w=self.shared)


def near_tie_tokens(logits64: np.ndarray, k: int, gap=TIE_GAP) -> np.ndarray:
    """R-17: flag tokens whose fp64 gap between two adjacent logits among the top-(k+1) is
    below `gap` but not zero.  An exact tie (gap 0) is not flagged: both sides then see equal
    logits and the lowest-id rule (R-3) decides, so the selection must match exactly."""
    s = -np.sort(-logits64, axis=1)[:, : k + 1]
    if s.shape[1] < 2:
        return np.zeros(logits64.shape[0], bool)
    d = np.abs(np.diff(s, axis=1))
    return ((d < gap) & (d > 0)).any(axis=1)


def rel_err(a, ref) -> float:
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    return float(np.abs(a - ref).max() / max(np.abs(ref).max(), 1e-30))


def to_np_f64(t: torch.Tensor) -> np.ndarray:
    return t.detach().float().cpu().numpy().astype(np.float64)


def check_routing(gpu_topk: np.ndarray, ref_logits: np.ndarray, ref_topk: np.ndarray, k: int):
    """Bit-exact top-k except on flagged near-tie tokens.  Returns the flag mask."""
    flagged = near_tie_tokens(ref_logits, k)
    bad = (~flagged) & (gpu_topk != ref_topk).any(axis=1)
    assert not bad.any(), f"unflagged routing mismatch on tokens {np.nonzero(bad)[0][:10]}"
    return flagged
