"""The certified tensor-core gate (gate_tc.cu) against the fp64 oracle and the fp64 DMMA gate.

Routing (expert ids, slots, drops, capacity) must be bit-exact (north_star): certified tokens
through the error bound, the rest re-decided from fp64 logits. Inputs here are adversarial:
exact logit ties (duplicated router columns, zero tokens), near-ties below the bound (columns
differing by 1 ulp-scale perturbations), and plain random rows. Reference: gate_linear +
softmax_rows + topk_select + assign_locations, gating.cpp:19-112."""
import numpy as np
import pytest
import torch

import oracle
from paper_2206_03382_b200 import LayerState, MoELayerConfig, forward
from paper_2206_03382_b200 import rng

pytestmark = pytest.mark.gpu


def _route(x, wg, E, k, f, M, T, precision, cap="fixed"):
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=256, tokens_per_step=T,
                         top_k=k, capacity=cap, capacity_factor=f, dtype="bf16",
                         gate_precision=precision)
    st = LayerState.init(cfg, 5)
    st.set_router(wg)
    forward(st, torch.as_tensor(x).to(torch.bfloat16).cuda())
    torch.cuda.synchronize()
    idxs, loc, gates, cap = st.routing()
    m = st.metrics()
    st.close()
    return idxs, loc, gates, cap, m


def _check_gates(gates, ref, x, wg):
    """Certified tokens' gate values carry the logits' fp32-accumulation error: relative to the
    fp64 gate, |dg / g| <= 2^-18 |x_t|_2 max_e |Wg[:, e]|_2 (typical errors are ~100x smaller;
    the certificate's own eps is 2^-14 |x| |w|). Re-decided tokens match to fp64 summation order."""
    bound = 2.0 ** -18 * np.linalg.norm(x, axis=1) * np.linalg.norm(wg, axis=0).max()
    with np.errstate(divide="ignore", invalid="ignore"):
        rel = np.where(gates == ref, 0.0, np.abs(gates - ref) / np.abs(ref)).max(axis=1)
    assert (rel <= np.maximum(bound, 1e-12)).all(), (rel.max(), bound.min())


def _inputs(seed, T, M, E, kind):
    x = rng.round_bf16(rng.uniform(seed, 0, T * M).reshape(T, M))
    wg = rng.uniform(seed, T * M, M * E).reshape(M, E)
    if kind == "dup_columns":       # experts 1 == 5 and 2 == 3: exact ties on every token
        wg[:, 5] = wg[:, 1]
        wg[:, 3] = wg[:, 2]
    elif kind == "near_ties":       # columns 4 / 6 differ by ~1e-9: ties far below the bound
        wg[:, 6] = wg[:, 4] * (1.0 + 1e-9)
        wg[:, 7] = wg[:, 0] + 3e-12
    elif kind == "zero_tokens":     # uniform softmax rows: every expert ties
        x[::7] = 0.0
    elif kind == "scaled":          # large logits: peaked softmax, tiny gaps relative to scale
        x *= 64.0
    return x, wg


@pytest.mark.parametrize("kind", ["random", "dup_columns", "near_ties", "zero_tokens", "scaled"])
@pytest.mark.parametrize("E,k,f", [(32, 1, 1.0), (16, 2, 1.25), (8, 4, 0.75)])
def test_certified_gate_routing_bit_exact(cuda, kind, E, k, f):
    T, M = 2048, 512
    x, wg = _inputs(17, T, M, E, kind)
    idxs, loc, gates, cap, m = _route(x, wg, E, k, f, M, T, "auto")
    probs = oracle.gate_linear(x, wg)
    r_idx, r_gates, r_loc, r_cap = oracle.run_gating_blocked(probs, 1, k, 0, f, False)
    assert cap == r_cap
    assert np.array_equal(idxs, r_idx), kind
    assert np.array_equal(loc, r_loc), kind
    _check_gates(gates, r_gates, x, wg)
    if kind in ("dup_columns", "zero_tokens"):
        assert m.gate_fixups > 0   # exact ties can never certify: the fp64 path decided them
    # the fp64 DMMA gate decides identically
    i2, l2, g2, c2, m2 = _route(x, wg, E, k, f, M, T, "fp64")
    assert np.array_equal(i2, idxs) and np.array_equal(l2, loc) and c2 == cap
    assert m2.gate_fixups == 0


def test_certified_gate_tgt_shape_fixup_rate(cuda):
    """TGT routing shape (32K tokens, M = 1024, E = 32): bit-exact and only a small fraction of
    tokens needs the fp64 re-decision."""
    T, M, E = 32768, 1024, 32
    x, wg = _inputs(402, T, M, E, "random")
    idxs, loc, gates, cap, m = _route(x, wg, E, 1, 1.0, M, T, "auto")
    probs = oracle.gate_linear(x, wg)
    r_idx, r_gates, r_loc, r_cap = oracle.run_gating_blocked(probs, 1, 1, 0, 1.0, False)
    assert np.array_equal(idxs, r_idx) and np.array_equal(loc, r_loc) and cap == r_cap
    _check_gates(gates, r_gates, x, wg)
    print("gate_fixups", m.gate_fixups, "max rel gate err", float(np.abs(gates / r_gates - 1).max()))
    assert 0 < m.gate_fixups < T // 10


@pytest.mark.parametrize("cap,kind,f", [("auto", 1, 1.0), ("bounded", 2, 1.25), ("bounded", 2, 0.5)])
def test_certified_gate_capacity_policies(cuda, cap, kind, f):
    """Auto / Bounded capacity (resolve_capacity, core.cpp:47-59) after the certified gate: the
    histograms the fix-up patched feed the capacity scan."""
    T, M, E, k = 3000, 512, 32, 2
    x, wg = _inputs(23, T, M, E, "near_ties")
    idxs, loc, gates, capv, m = _route(x, wg, E, k, f, M, T, "auto", cap)
    probs = oracle.gate_linear(x, wg)
    r_idx, r_gates, r_loc, r_cap = oracle.run_gating_blocked(probs, 1, k, kind, f, False)
    assert capv == r_cap
    assert np.array_equal(idxs, r_idx) and np.array_equal(loc, r_loc)
    assert m.drop_count == int((r_loc < 0).sum())
