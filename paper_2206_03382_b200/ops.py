"""Reference sub-operators (gating.hpp, dispatch.hpp, parallelism.hpp) on torch CUDA tensors.

Each call runs the sm_100a kernels of libmoe_b200.so on the current torch stream; shapes and
semantics follow the reference functions cited per wrapper. Used by the parity tests and
available for composing a layer by hand.
"""
from __future__ import annotations

import ctypes as C

import torch

from . import _lib
from ._lib import check, lib

_DT = {torch.bfloat16: _lib.DTYPE_BF16, torch.float32: _lib.DTYPE_F32, torch.float64: _lib.DTYPE_F64}
_CAP = {"fixed": _lib.CAP_FIXED, "auto": _lib.CAP_AUTO, "bounded": _lib.CAP_BOUNDED}


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _st(t):
    return C.c_void_p(torch.cuda.current_stream(t.device).cuda_stream)


def _need(t, name):
    if not (t.is_cuda and t.is_contiguous()):
        raise _lib.MoeError(_lib.MOE_EINVAL, f"{name} must be a contiguous CUDA tensor")


def gating(x: torch.Tensor, wg: torch.Tensor, blocks: int, k: int, capacity: str = "fixed",
           factor: float = 1.0, bpr: bool = False, want_probs: bool = False):
    """gate_linear + run_gating_blocked (gating.cpp:29-35, 134-162).

    x (blocks*T, M) bf16/f32, wg (M, E) fp64 -> idxs int32, gates fp64, locations int32 (n, k),
    capacity, drops, probs (n, E) or None."""
    _need(x, "x"); _need(wg, "wg")
    n, M = x.shape
    E = wg.shape[1]
    if n % blocks:
        raise _lib.MoeError(_lib.MOE_EINVAL, "run_gating_blocked: rows must split into equal blocks")
    T = n // blocks
    dev = x.device
    idxs = torch.empty(n, k, dtype=torch.int32, device=dev)
    gates = torch.empty(n, k, dtype=torch.float64, device=dev)
    loc = torch.empty(n, k, dtype=torch.int32, device=dev)
    probs = torch.empty(n, E, dtype=torch.float64, device=dev) if want_probs else None
    cap, drops = C.c_int64(), C.c_int64()
    check(lib().moe_op_gating(_p(x), _DT[x.dtype], _p(wg), blocks, T, M, E, k, _CAP[capacity],
                              float(factor), int(bpr), _p(idxs), _p(gates), _p(loc), _p(probs),
                              C.byref(cap), C.byref(drops), _st(x)))
    return idxs, gates, loc, cap.value, drops.value, probs


def gating_cosine(x: torch.Tensor, proj: torch.Tensor, experts: torch.Tensor, blocks: int, k: int,
                  temperature: float = 1.0, capacity: str = "fixed", factor: float = 1.0,
                  bpr: bool = False, want_probs: bool = False):
    """gate_cosine + run_gating_blocked (gating.cpp:37-56, 134-162): proj (M, D), experts (E, D)
    fp64; same outputs as gating()."""
    _need(x, "x"); _need(proj, "proj"); _need(experts, "experts")
    n, M = x.shape
    E, D = experts.shape
    if n % blocks:
        raise _lib.MoeError(_lib.MOE_EINVAL, "run_gating_blocked: rows must split into equal blocks")
    T = n // blocks
    dev = x.device
    idxs = torch.empty(n, k, dtype=torch.int32, device=dev)
    gates = torch.empty(n, k, dtype=torch.float64, device=dev)
    loc = torch.empty(n, k, dtype=torch.int32, device=dev)
    probs = torch.empty(n, E, dtype=torch.float64, device=dev) if want_probs else None
    cap, drops = C.c_int64(), C.c_int64()
    check(lib().moe_op_gating_cosine(_p(x), _DT[x.dtype], _p(proj), _p(experts), D,
                                     float(temperature), blocks, T, M, E, k, _CAP[capacity],
                                     float(factor), int(bpr), _p(idxs), _p(gates), _p(loc),
                                     _p(probs), C.byref(cap), C.byref(drops), _st(x)))
    return idxs, gates, loc, cap.value, drops.value, probs


def encode(x, blocks, E, k, capacity, degree, idxs, locations):
    """fast_encode_range per block + partition_capacity -> (blocks, degree, E, cc, M)."""
    _need(x, "x")
    n, M = x.shape
    T = n // blocks
    cc = -(-capacity // degree)
    z = torch.empty(blocks, degree, E, cc, M, dtype=x.dtype, device=x.device)
    check(lib().moe_op_encode(_p(x), _DT[x.dtype], blocks, T, M, E, k, capacity, degree,
                              _p(idxs), _p(locations), _p(z), _st(x)))
    return z


def decode(z, blocks, T, k, capacity, idxs, locations, gates):
    """fast_decode_range (dispatch.cpp:75-87); z (blocks, degree, E, cc, M)."""
    _need(z, "z")
    _, degree, E, cc, M = z.shape
    y = torch.empty(blocks * T, M, dtype=z.dtype, device=z.device)
    check(lib().moe_op_decode(_p(z), _DT[z.dtype], blocks, T, M, E, k, capacity, degree,
                              _p(idxs), _p(locations), _p(gates), _p(y), _st(z)))
    return y


def decode_backward(dy, z, blocks, E, k, capacity, degree, idxs, locations, gates,
                    want_dgates=False):
    """fast_decode_backward_range (dispatch.cpp:136-157) -> dz (blocks, degree, E, cc, M), dgates."""
    _need(dy, "dy")
    n, M = dy.shape
    T = n // blocks
    cc = -(-capacity // degree)
    dz = torch.empty(blocks, degree, E, cc, M, dtype=dy.dtype, device=dy.device)
    dg = torch.empty(n, k, dtype=torch.float64, device=dy.device) if want_dgates else None
    check(lib().moe_op_decode_backward(_p(dy), _p(z), _DT[dy.dtype], blocks, T, M, E, k, capacity,
                                       degree, _p(idxs), _p(locations), _p(gates), _p(dz), _p(dg),
                                       _st(dy)))
    return dz, dg


def encode_backward(dz, blocks, T, k, capacity, idxs, locations):
    """fast_encode_backward_range (dispatch.cpp:117-128)."""
    _need(dz, "dz")
    _, degree, E, cc, M = dz.shape
    dx = torch.empty(blocks * T, M, dtype=dz.dtype, device=dz.device)
    check(lib().moe_op_encode_backward(_p(dz), _DT[dz.dtype], blocks, T, M, E, k, capacity, degree,
                                       _p(idxs), _p(locations), _p(dx), _st(dz)))
    return dx


def expert_ffn(x, w1, w2, want_act=False):
    """expert_ffn (parallelism.cpp:103-121): x (n, rows, M), w1 (n, M, V), w2 (n, V, M)."""
    n, rows, M = x.shape
    V = w1.shape[2]
    y = torch.empty_like(x)
    act = torch.empty(n, rows, V, dtype=x.dtype, device=x.device) if want_act else None
    check(lib().moe_op_expert_ffn(_p(x), _p(w1), _p(w2), _p(y), _p(act), _DT[x.dtype], n, rows,
                                  M, V, _st(x)))
    return (y, act) if want_act else y


def expert_ffn_backward(x, w1, w2, dy):
    """expert_ffn_backward (parallelism.cpp:123-147) -> dx, dw1 (fp32), dw2 (fp32)."""
    n, rows, M = x.shape
    V = w1.shape[2]
    dx = torch.empty_like(x)
    dw1 = torch.empty(n, M, V, dtype=torch.float32, device=x.device)
    dw2 = torch.empty(n, V, M, dtype=torch.float32, device=x.device)
    check(lib().moe_op_expert_ffn_backward(_p(x), _p(w1), _p(w2), _p(dy), _p(dx), _p(dw1),
                                           _p(dw2), _DT[x.dtype], n, rows, M, V, _st(x)))
    return dx, dw1, dw2


def fill_uniform(out: torch.Tensor, seed: int, offset: int, lo: float = -1.0, hi: float = 1.0):
    """Rng(seed) draws offset.. on the device (core.cpp:66-83), rounded to out.dtype."""
    _need(out, "out")
    check(lib().moe_op_fill_uniform(_p(out), _DT[out.dtype], out.numel(), C.c_uint64(seed),
                                    C.c_uint64(offset), float(lo), float(hi), _st(out)))
    return out


def weight_stats(w1: torch.Tensor):
    """ReLU-certificate weight statistics of w1 [n][M][V] bf16 -> (colnorm [n][V] fp32,
    colnorm_blk [n][V/64] fp32, w1t [n][V][M] bf16)."""
    _need(w1, "w1")
    n, M, V = w1.shape
    colnorm = torch.empty(n, V, dtype=torch.float32, device=w1.device)
    blk = torch.empty(n * (V // 64) + 1, dtype=torch.float32, device=w1.device)  # [n][V/64]
    w1t = torch.empty(n, V, M, dtype=w1.dtype, device=w1.device)
    check(lib().moe_op_weight_stats(_p(w1), n, M, V, C.cast(_p(colnorm), _lib.PF),
                                    C.cast(_p(blk), _lib.PF), _p(w1t), _st(w1)))
    return colnorm, blk[:n * (V // 64)].view(n, V // 64), w1t
