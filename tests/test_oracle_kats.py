"""The CPU oracle pinned against the reference's own known-answer tests and properties
(tests/golden/reference_kats.json, transcribed with file:line). CPU only."""
import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_2206_03382_b200 import rng

KATS = json.loads((Path(__file__).parent / "golden" / "reference_kats.json").read_text())


def test_expert_capacity_kats():
    for c in KATS["expert_capacity"]:
        assert oracle.expert_capacity(c["k"], c["f"], c["T"], c["E"]) == c["cap"], c["src"]
    for c in KATS["expert_capacity_invalid"]:
        assert oracle.expert_capacity(c["k"], c["f"], c["T"], c["E"]) == -1, c["src"]


def test_resolve_capacity_kats():
    for c in KATS["resolve_capacity"]:
        assert oracle.resolve_capacity(c["kind"], c["factor"], c["demand"], c["E"], c["k"], c["T"]) == c["cap"], c["src"]


def test_capacity_factor_round_trip():
    c = KATS["capacity_factor_round_trip"]
    for f in c["fs"]:
        cap = oracle.expert_capacity(c["k"], f, c["T"], c["E"])
        back = oracle.capacity_to_factor(cap, c["E"], c["k"], c["T"])
        assert oracle.expert_capacity(c["k"], back, c["T"], c["E"]) == cap


def test_softmax_kats():
    for c in KATS["softmax"]:
        p = oracle.gate_linear(np.array(c["x"]), np.array(c["wg"]))
        np.testing.assert_allclose(p, np.array(c["probs"]), atol=1e-15)
        np.testing.assert_allclose(p.sum(axis=1), 1.0, atol=1e-12)


def test_topk_kats():
    for c in KATS["topk"]:
        idxs, gates = oracle.topk_select(np.array(c["probs"]), c["k"])
        assert idxs.tolist() == c["idxs"], c["src"]
        assert gates[0, 0] == c["gate00"]


def test_assign_locations_kats():
    for c in KATS["assign_locations"]:
        loc = oracle.assign_locations(np.array(c["idxs"]).reshape(-1, 1),
                                      np.array(c["gates"]).reshape(-1, 1), c["cap"], c["bpr"])
        assert loc[:, 0].tolist() == c["locations"], c["src"]


def test_run_gating_kats():
    for c in KATS["run_gating"]:
        idxs, gates, loc, cap = oracle.run_gating_blocked(np.array(c["probs"]), c["blocks"], c["k"],
                                                          c["kind"], c["factor"] or 1.0, False)
        assert cap == c["cap"], c["src"]
        if "drops" in c:
            assert int((loc < 0).sum()) == c["drops"]
        if "locations" in c:
            assert loc[:, 0].tolist() == c["locations"]


def test_encode_kat_and_dense_equivalence():
    c = KATS["encode"][0]
    idxs = np.array(c["idxs"]).reshape(-1, 1)
    loc = np.array(c["locations"]).reshape(-1, 1)
    z = oracle.encode(np.array(c["x"]), 1, c["E"], 1, c["cap"], idxs, loc)
    assert z[0].tolist() == c["z"]
    # random instances: sparse == dense einsum exactly, decode ~ dense (test_dispatch.cpp:48-77)
    r = np.random.RandomState(42)
    for i in range(40):
        T, E, M = r.randint(1, 25), r.randint(1, 9), r.randint(1, 9)
        k = r.randint(1, min(2, E) + 1)
        f = r.uniform(0.2, 1.5)
        probs = r.uniform(size=(T, E)) + 1e-3
        probs /= probs.sum(axis=1, keepdims=True)
        idxs, gates, loc, cap = oracle.run_gating_blocked(probs, 1, k, 0, f, i % 2 == 0)
        x = r.uniform(-1, 1, size=(T, M))
        z = oracle.encode(x, 1, E, k, cap, idxs, loc)
        assert np.array_equal(z[0], oracle.encode_dense(x, E, k, cap, idxs, loc))
        ze = r.uniform(-1, 1, size=(1, E, cap, M))
        y = oracle.decode(ze, 1, T, k, idxs, loc, gates)
        assert oracle.max_rel_diff(y, oracle.decode_dense(ze[0], T, k, idxs, loc, gates)) <= 1e-12


def test_dispatch_adjoint_and_fd():
    """Encode backward is the exact adjoint of encode; decode backward matches FD
    (test_dispatch.cpp:112-157)."""
    r = np.random.RandomState(45)
    T, E, M, k = 12, 4, 5, 2
    probs = r.uniform(size=(T, E)) + 1e-3
    probs /= probs.sum(axis=1, keepdims=True)
    idxs, gates, loc, cap = oracle.run_gating_blocked(probs, 1, k, 0, 0.8, False)
    x = r.uniform(-1, 1, (T, M))
    z = oracle.encode(x, 1, E, k, cap, idxs, loc)
    dz = r.uniform(-1, 1, z.shape)
    dx = oracle.encode_backward(dz, 1, T, k, idxs, loc)
    assert math.isclose((z * dz).sum(), (x * dx).sum(), rel_tol=1e-12)
    dy = r.uniform(-1, 1, (T, M))
    g_dz, g_dg = oracle.decode_backward(dy, z, 1, E, k, cap, idxs, loc, gates)
    h = 1e-6
    for i in range(0, z.size, 3):
        zp, zm = z.copy().ravel(), z.copy().ravel()
        zp[i] += h
        zm[i] -= h
        fd = ((oracle.decode(zp.reshape(z.shape), 1, T, k, idxs, loc, gates) * dy).sum() -
              (oracle.decode(zm.reshape(z.shape), 1, T, k, idxs, loc, gates) * dy).sum()) / (2 * h)
        assert g_dz.ravel()[i] == pytest.approx(fd, rel=1e-5, abs=1e-8)
    for t in range(T):
        for j in range(k):
            if loc[t, j] < 0:
                continue
            gp, gm = gates.copy(), gates.copy()
            gp[t, j] += h
            gm[t, j] -= h
            fd = ((oracle.decode(z, 1, T, k, idxs, loc, gp) * dy).sum() -
                  (oracle.decode(z, 1, T, k, idxs, loc, gm) * dy).sum()) / (2 * h)
            assert g_dg[t, j] == pytest.approx(fd, rel=1e-5, abs=1e-8)


def test_expert_ffn_kats_and_fd():
    for c in KATS["expert_ffn"]:
        y = oracle.expert_ffn(np.array(c["x"]), np.array(c["w1"]), np.array(c["w2"]))
        assert y.tolist() == c["y"], c["src"]
    r = np.random.RandomState(7)
    x = r.uniform(-1, 1, (1, 3, 2))
    w1 = r.uniform(-1, 1, (1, 2, 4))
    w2 = r.uniform(-1, 1, (1, 4, 2))
    dy = r.uniform(-1, 1, (1, 3, 2))
    dx, dw1, dw2 = oracle.expert_ffn_backward(x, w1, w2, dy)
    h = 1e-6
    loss = lambda xx, a, b: (oracle.expert_ffn(xx, a, b) * dy).sum()  # noqa: E731
    for arr, grad, idx in ((x, dx, 0), (w1, dw1, 1), (w2, dw2, 2)):
        for i in range(arr.size):
            p, m = arr.copy().ravel(), arr.copy().ravel()
            p[i] += h
            m[i] -= h
            args_p = [x, w1, w2]
            args_m = [x, w1, w2]
            args_p[idx] = p.reshape(arr.shape)
            args_m[idx] = m.reshape(arr.shape)
            fd = (loss(*args_p) - loss(*args_m)) / (2 * h)
            assert grad.ravel()[i] == pytest.approx(fd, rel=1e-5, abs=1e-7)


def test_partition_and_flex_layout_kats():
    c = KATS["partition_capacity"]
    x = np.random.RandomState(301).uniform(-1, 1, (c["E"], c["C"], c["M"]))
    ch = oracle.partition_capacity(x, c["degree"])
    assert ch.shape == (c["degree"], c["E"], c["cc"], c["M"])
    assert np.array_equal(ch[0, :, :2], x[:, :2]) and np.array_equal(ch[1, :, 0], x[:, 2])
    assert (ch[1, :, 1] == 0).all()
    assert np.array_equal(oracle.merge_chunks(ch, c["C"]), x)
    assert np.array_equal(oracle.merge_chunks(oracle.partition_capacity(x, 8), c["C"]), x)
    f = KATS["flex_all2all"]
    W, E, dC, M = f["W"], f["E"], f["dC"], f["M"]
    inp = np.random.RandomState(103).uniform(-1, 1, (W, E, dC, M))
    out = oracle.flex_dispatch(inp, W)
    dE = E // W
    for d in range(W):
        for e in range(dE):
            for r_ in range(W):
                assert np.array_equal(out[d, e, r_ * dC:(r_ + 1) * dC], inp[r_, d * dE + e])
    assert np.array_equal(oracle.flex_combine(out, W), inp)


def test_rng_matches_reference_stream():
    c = KATS["rng"]
    a = oracle.fill_uniform(c["seed"], 0, c["n"], 0.0, 1.0)
    assert ((a >= 0) & (a < 1)).all()
    assert np.array_equal(a, rng.uniform(c["seed"], 0, c["n"], 0.0, 1.0))
    # splitmix64 first outputs for seed 0 (public splitmix64 reference values)
    import ctypes as C
    s = C.c_uint64(0)
    first = [oracle.lib().orc_next_u64(C.byref(s)) for _ in range(3)]
    assert first == [0xE220A8397B1DCDAF, 0x6E789E6AA1B965F4, 0x06C45D188009454F]


def test_layer_oracle_matches_frozen_plan():
    """Blocked layer (W source blocks, gathered capacity) == per-token oracle
    (test_moe_layer.cpp:37-80), incl. top-2 BPR with drops."""
    for W, E, k, f, bpr in ((2, 4, 1, 1.0, False), (4, 8, 2, 0.5, True), (2, 4, 2, 1.25, True)):
        T, M, V = 4, 3, 8
        wg, w1, w2 = rng.layer_params(402, M, E, V)
        off = rng.draw_offsets(M, E, V, W, T)
        x = rng.uniform(402, off["x"], W * T * M).reshape(W * T, M)
        out = oracle.layer_step(x, wg, w1, w2, None, W, k, 0, f, bpr)
        want = oracle.frozen_plan_forward(x, k, out["idxs"], out["locations"], out["gates"], w1, w2)
        assert oracle.max_rel_diff(out["y"], want) <= 1e-12


def test_layer_oracle_backward_fd():
    """Whole-layer backward vs central differences with the plan frozen (test_moe_layer.cpp:154-200)."""
    W, E, k, T, M, V = 2, 4, 1, 3, 2, 4
    wg, w1, w2 = rng.layer_params(410, M, E, V)
    off = rng.draw_offsets(M, E, V, W, T)
    x = rng.uniform(410, off["x"], W * T * M).reshape(W * T, M)
    dy = rng.uniform(410, off["dy"], W * T * M).reshape(W * T, M)
    out = oracle.layer_step(x, wg, w1, w2, dy, W, k)
    plan = (out["idxs"], out["locations"], out["gates"])
    h = 1e-6

    def loss(xx, a, b):
        return (oracle.frozen_plan_forward(xx, k, *plan, a, b) * dy).sum()
    for i in range(0, x.size, 3):
        p, m = x.copy().ravel(), x.copy().ravel()
        p[i] += h
        m[i] -= h
        fd = (loss(p.reshape(x.shape), w1, w2) - loss(m.reshape(x.shape), w1, w2)) / (2 * h)
        assert out["dx"].ravel()[i] == pytest.approx(fd, rel=1e-5, abs=1e-7)
    for i in range(0, w1.size, 3):
        p, m = w1.copy().ravel(), w1.copy().ravel()
        p[i] += h
        m[i] -= h
        fd = (loss(x, p.reshape(w1.shape), w2) - loss(x, m.reshape(w1.shape), w2)) / (2 * h)
        assert out["dw1"].ravel()[i] == pytest.approx(fd, rel=1e-5, abs=1e-7)


def test_bf16_rounding_is_nearest_even():
    """Direct fp64 -> bf16 round-to-nearest-even (no double rounding through fp32): check against
    the two bracketing bf16 values computed exactly."""
    x = np.concatenate([rng.uniform(5, 0, 100000, -3, 3),
                        1.0 + np.array([2.0 ** -8, 3 * 2.0 ** -8, 2.0 ** -8 + 2.0 ** -30])])
    u = x.view(np.uint64)
    lo = (u & ~np.uint64((1 << 45) - 1)).view(np.float64)          # truncate toward zero
    hi = (((u >> np.uint64(45)) + np.uint64(1)) << np.uint64(45)).view(np.float64)
    dlo, dhi = np.abs(x - lo), np.abs(hi - x)
    lo_even = ((u >> np.uint64(45)) & np.uint64(1)) == 0
    want = np.where(dlo < dhi, lo, np.where(dhi < dlo, hi, np.where(lo_even, lo, hi)))
    assert np.array_equal(rng.round_bf16(x), want)


def test_cosine_gate_kat():
    """test_gating.cpp:38-53: the temperature clamps at 0.01, rows sum to 1, a zero-norm expert
    row is rejected (invalid_argument)."""
    rng = np.random.default_rng(13)
    x = rng.uniform(-1, 1, (4, 3))
    proj = rng.uniform(-1, 1, (3, 6))
    experts = rng.uniform(-1, 1, (5, 6))
    p = oracle.gate_cosine(x, proj, experts, 1e-9)
    p2 = oracle.gate_cosine(x, proj, experts, 0.01)
    assert np.abs(p - p2).max() == 0.0
    np.testing.assert_allclose(p.sum(axis=1), 1.0, rtol=1e-12)
    experts[2] = 0.0
    with pytest.raises(ValueError):
        oracle.gate_cosine(x, proj, experts, 1.0)
    # zero-norm projected token (x row of zeros) is rejected as well (gating.cpp:46-47)
    experts[2] = 1.0
    x[1] = 0.0
    with pytest.raises(ValueError):
        oracle.gate_cosine(x, proj, experts, 1.0)


def test_layer_step_sharded_placement_matches_frozen_plan():
    """E < W (RanksPerExpert): the oracle's layer equals the per-token frozen plan
    (frozen_plan_forward, moe_layer.cpp:321-335) -- placement changes who computes, not what."""
    import numpy as np
    import oracle
    from tests.helpers import layer_inputs
    for W, E, k in ((4, 2, 1), (4, 2, 2), (2, 1, 1)):
        T, M, V = 16, 8, 16
        inp = layer_inputs(402, W, T, M, V, E, "f32")
        ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], W, k, 0, 1.0, False)
        y = np.zeros_like(inp["x"])
        for t in range(W * T):
            for j in range(k):
                if ref["locations"][t, j] < 0:
                    continue
                e = ref["idxs"][t, j]
                h = np.maximum(inp["x"][t] @ inp["w1"][e], 0.0)
                y[t] += ref["gates"][t, j] * (h @ inp["w2"][e])
        assert oracle.max_rel_diff(y, ref["y"]) < 1e-12
        assert np.abs(ref["dw1"]).max() > 0 and np.abs(ref["dx"]).max() > 0


@pytest.mark.parametrize("W,k,f,bpr", [(2, 1, 1.0, False), (2, 2, 0.75, True)])
def test_sampled_oracle_matches_whole_layer(W, k, f, bpr):
    """The sampled checkers used at full C4 size (frozen-plan backward rows; an expert's dW1
    columns / dW2 rows from its gathered rows) equal the whole-layer oracle on a small layer."""
    E, M, V, T = 4 * W, 24, 40, 64
    x = rng.uniform(7, 0, W * T * M).reshape(W * T, M)
    dy = rng.uniform(7, 10**6, W * T * M).reshape(W * T, M)
    wg, w1, w2 = rng.layer_params(7, M, E, V)
    ref = oracle.layer_step(x, wg, w1, w2, dy, W, k, 0, f, bpr)
    idxs, loc, gates = ref["idxs"], ref["locations"], ref["gates"]
    sel = np.array([0, 3, 17, T + 5, W * T - 1])
    dx = oracle.frozen_plan_backward_rows(x[sel], dy[sel], k, idxs[sel], loc[sel], gates[sel], w1, w2)
    assert oracle.max_rel_diff(dx, ref["dx"][sel]) < 1e-12
    cols = np.array([0, 7, V - 1])
    for e in range(E):
        t, j = np.nonzero((idxs == e) & (loc >= 0))
        X = x[t]
        dZ = gates[t, j][:, None] * dy[t]
        d1, d2 = oracle.expert_backward_columns(X, dZ, w1[e], w2[e], cols)
        assert oracle.max_rel_diff(d1, ref["dw1"][e][:, cols]) < 1e-12
        assert oracle.max_rel_diff(d2, ref["dw2"][e][cols, :]) < 1e-12
