"""numpy/ctypes front-end of the fp64 CPU oracle (oracle/moe_oracle.c).

TEST INFRASTRUCTURE ONLY -- the parity checker and CPU baseline. Only tests/, __graft_entry__
.smoke() and bench.py's cpu_baseline / --impl reference leg may import this module. The product
package (paper_2206_03382_b200) never imports it and has no CPU fallback.

Parity status: pinned against the reference's own known-answer tests (values transcribed with
file:line into tests/golden/reference_kats.json and checked by tests/test_oracle_kats.py). The
reference itself cannot be compiled here (Eigen 3 and its vendored test deps are absent), so no
reference-generated fixtures exist; see DESIGN.md "Oracle".
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "liboracle.so"

_l = None


def build() -> Path:
    r = subprocess.run(["make", "-C", str(HERE), "CC=gcc"], capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")
    return LIB


def lib() -> C.CDLL:
    global _l
    if _l is None:
        if not LIB.exists():
            build()
        _l = C.CDLL(str(LIB))
        _l.orc_expert_capacity.restype = C.c_int64
        _l.orc_resolve_capacity.restype = C.c_int64
        _l.orc_capacity_to_factor.restype = C.c_double
        _l.orc_run_gating_blocked.restype = C.c_int64
        _l.orc_drop_count.restype = C.c_int64
        _l.orc_layer_step.restype = C.c_int64
        _l.orc_layer_step_probs.restype = C.c_int64
        _l.orc_gate_cosine.restype = C.c_int32
        _l.orc_num_threads.restype = C.c_int32
        _l.orc_next_u64.restype = C.c_uint64
        _l.orc_uniform.restype = C.c_double
    return _l


def _p(a: np.ndarray | None):
    if a is None:
        return None
    assert a.flags["C_CONTIGUOUS"], "oracle arrays must be C-contiguous"
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


I64, D = C.c_int64, C.c_double


def num_threads() -> int:
    return int(lib().orc_num_threads())


def set_num_threads(n: int) -> None:
    lib().orc_set_num_threads(C.c_int32(n))


def fill_uniform(seed: int, offset: int, n: int, lo: float, hi: float) -> np.ndarray:
    out = np.empty(n, np.float64)
    lib().orc_fill_uniform(C.c_uint64(seed), C.c_uint64(offset), I64(n), D(lo), D(hi), _p(out))
    return out


def expert_capacity(k, f, tokens, experts) -> int:
    return int(lib().orc_expert_capacity(I64(k), D(f), I64(tokens), I64(experts)))


def resolve_capacity(kind, factor, demand, E, k, T) -> int:
    d = _i64(demand)
    return int(lib().orc_resolve_capacity(C.c_int32(kind), D(factor), _p(d), I64(E), I64(k), I64(T)))


def capacity_to_factor(cap, E, k, T) -> float:
    return float(lib().orc_capacity_to_factor(I64(cap), I64(E), I64(k), I64(T)))


def gate_linear(x, wg) -> np.ndarray:
    x, wg = _f64(x), _f64(wg)
    T, M = x.shape
    E = wg.shape[1]
    out = np.empty((T, E), np.float64)
    lib().orc_gate_linear(_p(x), _p(wg), I64(T), I64(M), I64(E), _p(out))
    return out


def gate_cosine(x, proj, experts, temperature=1.0) -> np.ndarray:
    """gating.cpp:37-56; raises ValueError on a zero-norm token / expert (invalid_argument)."""
    x, proj, experts = _f64(x), _f64(proj), _f64(experts)
    T, M = x.shape
    E, Dd = experts.shape
    out = np.empty((T, E), np.float64)
    rc = lib().orc_gate_cosine(_p(x), _p(proj), _p(experts), D(temperature), I64(T), I64(M),
                               I64(E), I64(Dd), _p(out))
    if rc != 0:
        raise ValueError("gate_cosine: zero-norm projected token or expert row")
    return out


def topk_select(probs, k):
    probs = _f64(probs)
    T, E = probs.shape
    idxs = np.empty((T, k), np.int64)
    gates = np.empty((T, k), np.float64)
    lib().orc_topk_select(_p(probs), I64(T), I64(E), I64(k), _p(idxs), _p(gates))
    return idxs, gates


def assign_locations(idxs, gates, cap, bpr):
    idxs, gates = _i64(idxs), _f64(gates)
    T, k = idxs.shape
    loc = np.empty((T, k), np.int64)
    lib().orc_assign_locations(_p(idxs), _p(gates), I64(T), I64(k), I64(cap), C.c_int32(int(bpr)),
                               _p(loc))
    return loc


def run_gating_blocked(probs, blocks, k, cap_kind, factor, bpr):
    """Returns (idxs, gates, locations, capacity); probs (blocks*T, E)."""
    probs = _f64(probs)
    n, E = probs.shape
    T = n // blocks
    idxs = np.empty((n, k), np.int64)
    gates = np.empty((n, k), np.float64)
    loc = np.empty((n, k), np.int64)
    cap = lib().orc_run_gating_blocked(_p(probs), I64(blocks), I64(T), I64(E), I64(k),
                                       C.c_int32(cap_kind), D(factor), C.c_int32(int(bpr)),
                                       _p(idxs), _p(gates), _p(loc))
    return idxs, gates, loc, int(cap)


def encode(x, blocks, E, k, cap, idxs, locations):
    x = _f64(x)
    n, M = x.shape
    T = n // blocks
    z = np.empty((blocks, E, cap, M), np.float64)
    lib().orc_encode(_p(x), I64(blocks), I64(T), I64(M), I64(E), I64(k), I64(cap),
                     _p(_i64(idxs)), _p(_i64(locations)), _p(z))
    return z


def decode(z, blocks, T, k, idxs, locations, gates):
    z = _f64(z)
    _, E, cap, M = z.shape
    y = np.empty((blocks * T, M), np.float64)
    lib().orc_decode(_p(z), I64(blocks), I64(T), I64(M), I64(E), I64(k), I64(cap),
                     _p(_i64(idxs)), _p(_i64(locations)), _p(_f64(gates)), _p(y))
    return y


def decode_backward(dy, z, blocks, E, k, cap, idxs, locations, gates, want_dgates=True):
    dy = _f64(dy)
    n, M = dy.shape
    T = n // blocks
    dz = np.empty((blocks, E, cap, M), np.float64)
    dg = np.empty((n, k), np.float64) if want_dgates else None
    zz = _f64(z) if z is not None else None
    lib().orc_decode_backward(_p(dy), _p(zz), I64(blocks), I64(T), I64(M), I64(E), I64(k),
                              I64(cap), _p(_i64(idxs)), _p(_i64(locations)), _p(_f64(gates)),
                              _p(dz), _p(dg))
    return dz, dg


def encode_backward(dz, blocks, T, k, idxs, locations):
    dz = _f64(dz)
    _, E, cap, M = dz.shape
    dx = np.empty((blocks * T, M), np.float64)
    lib().orc_encode_backward(_p(dz), I64(blocks), I64(T), I64(M), I64(E), I64(k), I64(cap),
                              _p(_i64(idxs)), _p(_i64(locations)), _p(dx))
    return dx


def encode_dense(x, E, k, cap, idxs, locations):
    x = _f64(x)
    T, M = x.shape
    z = np.empty((E, cap, M), np.float64)
    lib().orc_encode_dense(_p(x), I64(T), I64(M), I64(E), I64(k), I64(cap), _p(_i64(idxs)),
                           _p(_i64(locations)), _p(z))
    return z


def decode_dense(z, T, k, idxs, locations, gates):
    z = _f64(z)
    E, cap, M = z.shape
    y = np.empty((T, M), np.float64)
    lib().orc_decode_dense(_p(z), I64(T), I64(M), I64(E), I64(k), I64(cap), _p(_i64(idxs)),
                           _p(_i64(locations)), _p(_f64(gates)), _p(y))
    return y


def partition_capacity(x, degree):
    x = _f64(x)
    E, Cc, M = x.shape
    cc = -(-Cc // degree)
    out = np.empty((degree, E, cc, M), np.float64)
    lib().orc_partition_capacity(_p(x), I64(E), I64(Cc), I64(M), I64(degree), _p(out))
    return out


def merge_chunks(chunks, C_orig):
    chunks = _f64(chunks)
    d, E, cc, M = chunks.shape
    out = np.empty((E, C_orig, M), np.float64)
    lib().orc_merge_chunks(_p(chunks), I64(E), I64(cc), I64(M), I64(d), I64(C_orig), _p(out))
    return out


def flex_dispatch(inp, W):
    inp = _f64(inp)  # (W, E, dC, M)
    _, E, dC, M = inp.shape
    out = np.empty((W, E // W, W * dC, M), np.float64)
    lib().orc_flex_dispatch(_p(inp), I64(W), I64(E), I64(dC), I64(M), _p(out))
    return out


def flex_combine(inp, W):
    inp = _f64(inp)  # (W, dE, W*dC, M)
    _, dE, WdC, M = inp.shape
    dC = WdC // W
    out = np.empty((W, dE * W, dC, M), np.float64)
    lib().orc_flex_combine(_p(inp), I64(W), I64(dE * W), I64(dC), I64(M), _p(out))
    return out


def expert_ffn(x, w1, w2):
    x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
    n, rows, M = x.shape
    V = w1.shape[2]
    y = np.empty_like(x)
    lib().orc_expert_ffn(_p(x), _p(w1), _p(w2), I64(n), I64(rows), I64(M), I64(V), _p(y))
    return y


def expert_ffn_backward(x, w1, w2, dy):
    x, w1, w2, dy = _f64(x), _f64(w1), _f64(w2), _f64(dy)
    n, rows, M = x.shape
    V = w1.shape[2]
    dx = np.empty_like(x)
    dw1 = np.empty((n, M, V), np.float64)
    dw2 = np.empty((n, V, M), np.float64)
    lib().orc_expert_ffn_backward(_p(x), _p(w1), _p(w2), _p(dy), I64(n), I64(rows), I64(M),
                                  I64(V), _p(dx), _p(dw1), _p(dw2))
    return dx, dw1, dw2


def frozen_plan_forward(x, k, idxs, locations, gates, w1, w2):
    x, w1, w2 = _f64(x), _f64(w1), _f64(w2)
    T, M = x.shape
    V = w1.shape[2]
    y = np.empty_like(x)
    lib().orc_frozen_plan_forward(_p(x), I64(T), I64(M), I64(V), I64(k), _p(_i64(idxs)),
                                  _p(_i64(locations)), _p(_f64(gates)), _p(w1), _p(w2), _p(y))
    return y


def frozen_plan_backward_rows(x, dy, k, idxs, locations, gates, w1, w2):
    """dx of the listed tokens under a frozen plan (moe_layer.cpp:246-319); rows independent."""
    x, dy, w1, w2 = _f64(x), _f64(dy), _f64(w1), _f64(w2)
    T, M = x.shape
    V = w1.shape[2]
    dx = np.empty_like(x)
    lib().orc_frozen_plan_backward_rows(_p(x), _p(dy), I64(T), I64(M), I64(V), I64(k),
                                        _p(_i64(idxs)), _p(_i64(locations)), _p(_f64(gates)),
                                        _p(w1), _p(w2), _p(dx))
    return dx


def expert_backward_columns(X, dZ, w1, w2, cols):
    """dW1[:, cols] (M, n) and dW2[cols, :] (n, M) of one expert from its rows (X, dZ)."""
    X, dZ, w1, w2 = _f64(X), _f64(dZ), _f64(w1), _f64(w2)
    rows, M = X.shape
    V = w1.shape[1]
    cols = _i64(cols)
    n = cols.shape[0]
    dw1c = np.empty((M, n), np.float64)
    dw2r = np.empty((n, M), np.float64)
    lib().orc_expert_backward_columns(_p(X), _p(dZ), I64(rows), I64(M), I64(V), _p(w1), _p(w2),
                                      I64(n), _p(cols), _p(dw1c), _p(dw2r))
    return dw1c, dw2r


def layer_step(x, wg, w1, w2, dy, W, k, cap_kind=0, factor=1.0, bpr=False, cosine=None):
    """Whole layer over W source blocks; returns dict of y, routing and (if dy) dx, dw1, dw2.
    cosine = (proj (M, D), experts (E, D), temperature) selects RouterKind::Cosine."""
    x, wg, w1, w2 = _f64(x), _f64(wg), _f64(w1), _f64(w2)
    n, M = x.shape
    T = n // W
    E, _, V = w1.shape
    y = np.empty((n, M), np.float64)
    idxs = np.empty((n, k), np.int64)
    loc = np.empty((n, k), np.int64)
    gates = np.empty((n, k), np.float64)
    dyy = _f64(dy) if dy is not None else None
    dx = np.empty((n, M), np.float64) if dy is not None else None
    dw1 = np.empty((E, M, V), np.float64) if dy is not None else None
    dw2 = np.empty((E, V, M), np.float64) if dy is not None else None
    probs = gate_cosine(x, *cosine) if cosine is not None else gate_linear(x, wg)
    cap = lib().orc_layer_step_probs(_p(x), _p(probs), _p(w1), _p(w2), _p(dyy), I64(W), I64(T),
                                     I64(M), I64(V), I64(E), I64(k), C.c_int32(cap_kind),
                                     D(factor), C.c_int32(int(bpr)), _p(y), _p(idxs), _p(loc),
                                     _p(gates), _p(dx), _p(dw1), _p(dw2))
    return dict(y=y, idxs=idxs, locations=loc, gates=gates, capacity=int(cap), dx=dx, dw1=dw1,
                dw2=dw2)


def max_rel_diff(a, b) -> float:
    """tensor.cpp:52-55: max|a-b| / max(max|a|, max|b|, 1e-300)."""
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    scale = max(np.abs(a).max(initial=0.0), np.abs(b).max(initial=0.0), 1e-300)
    return float(np.abs(a - b).max(initial=0.0) / scale)
