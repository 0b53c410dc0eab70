"""Shared builders for parity tests: reference-recipe inputs (Rng draw order), GPU runs, oracle."""
from __future__ import annotations

import numpy as np

from paper_2206_03382_b200 import rng


def layer_inputs(seed, W, T, M, V, E, dtype="bf16", with_dy=True, experts=None):
    """LayerState::init draws + x, dy (test_moe_layer.cpp:70-73,172), rounded to the layer dtype
    exactly as the GPU receives them (the oracle is fed the same rounded values)."""
    off = rng.draw_offsets(M, E, V, W, T)
    wg, w1, w2 = rng.layer_params(seed, M, E, V, experts)
    x = rng.uniform(seed, off["x"], W * T * M).reshape(W * T, M)
    dy = rng.uniform(seed, off["dy"], W * T * M).reshape(W * T, M) if with_dy else None
    r = lambda a: rng.round_dtype(a, dtype)  # noqa: E731
    cp, ce = rng.cosine_params(seed, M, E)
    return dict(wg=wg, w1=r(w1), w2=r(w2), x=r(x), dy=r(dy) if with_dy else None,
                cos_proj=cp, cos_experts=ce)


def probs_to_inputs(probs):
    """(x, wg) such that softmax(x . wg) reproduces `probs` row-for-row (ties exactly preserved):
    x = identity (T x T), wg = log(probs)."""
    p = np.asarray(probs, np.float64)
    T = p.shape[0]
    return np.eye(T), np.log(p)


def row_probs(idx, gate, E):
    """A probability row whose top-1 is (idx, gate): the rest spread evenly (needs gate > rest)."""
    rest = (1.0 - gate) / (E - 1)
    assert gate > rest
    row = np.full(E, rest)
    row[idx] = gate
    return row
