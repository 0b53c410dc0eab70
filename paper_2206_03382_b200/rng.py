"""Host-side copy of the reference generator and dtype rounding (core.cpp:66-83).

splitmix64 is counter-based: call n (1-based) of Rng(seed).next_u64() is mix(seed + n*gamma),
so any slice of the LayerState::init draw sequence (moe_layer.cpp:144-163) can be produced
vectorised. The same stream is generated on the device by moe_op_fill_uniform / moe_init_params.
"""
from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
COSINE_DIM = 256  # kCosineProjDim, moe_layer.cpp:23


def uniform(seed: int, offset: int, n: int, lo: float = -1.0, hi: float = 1.0) -> np.ndarray:
    """Draws offset .. offset+n-1 of Rng(seed).uniform(lo, hi) as fp64."""
    with np.errstate(over="ignore"):
        idx = np.arange(offset + 1, offset + n + 1, dtype=np.uint64)
        z = np.uint64(seed) + idx * GAMMA
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        z = z ^ (z >> np.uint64(31))
    u = (z >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)
    return lo + (hi - lo) * u


def round_bf16(a: np.ndarray) -> np.ndarray:
    """Round fp64 -> nearest-even bf16, returned as fp64 (no double rounding via fp32)."""
    a = np.ascontiguousarray(a, np.float64)
    u = a.view(np.uint64).copy()
    finite = (u & np.uint64(0x7FF0000000000000)) != np.uint64(0x7FF0000000000000)
    lsb = (u >> np.uint64(45)) & np.uint64(1)
    r = (u + (np.uint64((1 << 44) - 1) + lsb)) & ~np.uint64((1 << 45) - 1)
    u = np.where(finite, r, u)
    return u.view(np.float64)


def round_dtype(a: np.ndarray, dtype: str) -> np.ndarray:
    if dtype == "bf16":
        return round_bf16(a)
    if dtype == "f32":
        return np.asarray(a, np.float64).astype(np.float32).astype(np.float64)
    return np.asarray(a, np.float64)


def draw_offsets(M: int, E: int, V: int, W: int, T: int) -> dict:
    """Index of the first draw of each LayerState::init tensor (moe_layer.cpp:144-163) and of the
    x / dy draws the reference tests make next (test_moe_layer.cpp:72-73, 172)."""
    wg = 0
    cos_proj = wg + M * E
    cos_exp = cos_proj + M * COSINE_DIM
    experts = cos_exp + E * COSINE_DIM
    x = experts + E * 2 * M * V
    dy = x + W * T * M
    return dict(wg=wg, cosine_proj=cos_proj, cosine_experts=cos_exp, experts=experts, x=x, dy=dy,
                expert_stride=2 * M * V)


def cosine_params(seed: int, M: int, E: int):
    """RouterParams cosine_proj (M, 256) and cosine_experts (E, 256) (moe_layer.cpp:154-160)."""
    off = draw_offsets(M, E, 1, 1, 1)
    proj = uniform(seed, off["cosine_proj"], M * COSINE_DIM).reshape(M, COSINE_DIM)
    experts = uniform(seed, off["cosine_experts"], E * COSINE_DIM).reshape(E, COSINE_DIM)
    return proj, experts


def layer_params(seed: int, M: int, E: int, V: int, experts=None):
    """Wg (M,E) fp64 and w1 (n,M,V), w2 (n,V,M) fp64 for the given global experts."""
    off = draw_offsets(M, E, V, 1, 1)
    wg = uniform(seed, off["wg"], M * E).reshape(M, E)
    experts = range(E) if experts is None else experts
    w1s, w2s = [], []
    for e in experts:
        o = off["experts"] + e * off["expert_stride"]
        w1s.append(uniform(seed, o, M * V, -0.5, 0.5).reshape(M, V))
        w2s.append(uniform(seed, o + M * V, V * M, -0.5, 0.5).reshape(V, M))
    return wg, np.stack(w1s), np.stack(w2s)
