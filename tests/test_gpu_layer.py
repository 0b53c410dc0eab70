"""Whole-layer parity (forward + backward) on one B200 against the fp64 oracle.

Tolerances per north_star, using the reference's max_rel_diff (tensor.cpp:52-55): 1e-5 for the
fp32 path, 2e-2 for the bf16 tensor-core path; routing bit-exact. Large configs check full
routing + the full outputs against the oracle's per-expert GEMM restatement.
"""
import numpy as np
import pytest
import torch

import oracle
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward
from tests.helpers import layer_inputs

pytestmark = pytest.mark.gpu

CASES = [
    # E, k, f, M, V, T, bpr, dtype
    ("C1", 8, 1, 1.0, 512, 2048, 4096, False, "f32"),        # configs[0] at full size
    ("tiny-f32", 4, 2, 0.5, 3, 8, 4, True, "f32"),           # reference-test scale, drops
    ("small-bf16-tc", 8, 2, 1.25, 256, 512, 512, True, "bf16"),
    ("small-bf16-simt", 6, 1, 1.0, 40, 72, 300, False, "bf16"),
    ("mid-bf16", 16, 1, 1.0, 512, 1024, 4096, False, "bf16"),
]


def run_case(E, k, f, M, V, T, bpr, dt, seed=402, dev=0, cap="fixed"):
    cfg = MoELayerConfig(world_size=1, global_experts=E, model_dim=M, hidden_dim=V,
                         tokens_per_step=T, top_k=k, capacity=cap, capacity_factor=f, bpr=bpr,
                         dtype=dt)
    inp = layer_inputs(seed, 1, T, M, V, E, dt)
    st = LayerState.init(cfg, seed)
    tdt = cfg.torch_dtype
    x = torch.as_tensor(inp["x"]).to(tdt).cuda()
    dy = torch.as_tensor(inp["dy"]).to(tdt).cuda()
    res = forward(st, x)
    g = backward(st, res.saved, dy)
    torch.cuda.synchronize()
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], 1, k, kind, f, bpr)
    return st, res, g, ref, inp


@pytest.mark.parametrize("case", CASES, ids=lambda c: c[0])
def test_layer_forward_backward(cuda, case):
    _, E, k, f, M, V, T, bpr, dt = case
    st, res, g, ref, _ = run_case(E, k, f, M, V, T, bpr, dt)
    idxs, loc, gates, cap = st.routing()
    assert cap == ref["capacity"]
    assert np.array_equal(idxs, ref["idxs"])
    assert np.array_equal(loc, ref["locations"])
    # gate values: fp64 DMMA gate (f32 / BPR layers) up to summation order; the certified
    # tensor-core gate (bf16 FIFO) carries its logit error -- ~1e-6 typical, checked at 1e-4
    certified = dt == "bf16" and not bpr and E % 8 == 0 and M % 64 == 0
    np.testing.assert_allclose(gates, ref["gates"], rtol=1e-4 if certified else 1e-12, atol=0)
    tol = 1e-5 if dt == "f32" else 2e-2
    y = res.y.double().cpu().numpy()
    assert oracle.max_rel_diff(y, ref["y"]) < tol
    dropped = (ref["locations"] < 0).all(axis=1)
    assert (y[dropped] == 0).all()   # dropped rows are exactly zero (test_moe_layer.cpp:135-152)
    assert oracle.max_rel_diff(g.dx.double().cpu().numpy(), ref["dx"]) < tol
    assert oracle.max_rel_diff(g.dw1.double().cpu().numpy(), ref["dw1"]) < tol
    assert oracle.max_rel_diff(g.dw2.double().cpu().numpy(), ref["dw2"]) < tol
    m = st.metrics()
    assert m.capacity == cap and m.drop_count == int((loc < 0).sum())
    # the SIMT fallback is reported (shape cliff): only where N % 256 / K % 64 rule out tcgen05
    tc_shape = dt == "bf16" and M % 256 == 0 and V % 256 == 0
    assert (m.simt_gemms == 0) == (tc_shape or dt == "f32")


@pytest.mark.parametrize("cap,f", [("auto", 1.0), ("bounded", 1.25), ("bounded", 0.5)])
def test_layer_auto_bounded_capacity(cuda, cap, f):
    """AutoCapacity / BoundedCapacity inside the layer (resolve_capacity, core.cpp:47-59): the
    capacity follows the step's max demand (Auto grows the buffers), routing stays bit-exact."""
    st, res, g, ref, _ = run_case(8, 2, f, 256, 512, 1024, True, "bf16", cap=cap)
    idxs, loc, gates, capv = st.routing()
    assert capv == ref["capacity"]
    assert np.array_equal(idxs, ref["idxs"]) and np.array_equal(loc, ref["locations"])
    if cap == "auto":
        assert (loc >= 0).all()  # Auto never drops
    for name, got in (("y", res.y), ("dx", g.dx), ("dw1", g.dw1), ("dw2", g.dw2)):
        assert oracle.max_rel_diff(got.double().cpu().numpy(), ref[name]) < 2e-2, name


def test_layer_deterministic(cuda):
    """Two identical runs are bit-identical (test_moe_layer.cpp:118-133)."""
    a = run_case(8, 2, 1.0, 256, 512, 1024, True, "bf16", seed=407)
    b = run_case(8, 2, 1.0, 256, 512, 1024, True, "bf16", seed=407)
    assert torch.equal(a[1].y, b[1].y)
    assert torch.equal(a[2].dx, b[2].dx)
    assert torch.equal(a[2].dw1, b[2].dw1) and torch.equal(a[2].dw2, b[2].dw2)


def test_layer_set_weights_matches_init(cuda):
    """Explicit router/expert upload (moe_set_router/moe_set_expert) == on-device init draw."""
    E, M, V, T = 4, 64, 256, 128
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=1)
    inp = layer_inputs(11, 1, T, M, V, E, "bf16")
    a = LayerState.init(cfg, 11)
    b = LayerState(cfg)
    b.set_router(inp["wg"])
    for e in range(E):
        b.set_expert(e, inp["w1"][e], inp["w2"][e])
    wa, wb = a.weights(), b.weights()
    assert torch.equal(wa[0], wb[0]) and torch.equal(wa[1], wb[1])
    x = torch.as_tensor(inp["x"]).to(torch.bfloat16).cuda()
    assert torch.equal(forward(a, x).y, forward(b, x).y)


def test_layer_slices_gather_single_rank(cuda):
    """ZeRO slice upload + gather (parallelism.cpp:149-206) reassembles the full experts."""
    E, M, V, T = 2, 32, 64, 16
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=1,
                         dtype="f32")
    inp = layer_inputs(5, 1, T, M, V, E, "f32")
    s = LayerState(cfg)
    s.set_expert_slices(inp["w1"], inp["w2"])  # W = 1: the slice is the whole expert
    w1, w2 = s.weights()
    assert np.array_equal(w1.double().cpu().numpy(), inp["w1"])
    assert np.array_equal(w2.double().cpu().numpy(), inp["w2"])


@pytest.mark.parametrize("keep_views", [False, True])
def test_in_place_weight_update(cuda, keep_views):
    """An on-device SGD step written through the exported weight pointers: the next
    forward must rebuild the ReLU certificate's W1^T copy and column norms, so y, dx and dW match
    the oracle run on the updated weights. keep_views: views fetched before the step, then
    moe_weights_updated; else views fetched after the step (the fetch marks the state stale)."""
    E, k, f, M, V, T = 8, 1, 1.0, 512, 1024, 4096
    st, res, g, _, inp = run_case(E, k, f, M, V, T, False, "bf16")
    dw1, dw2 = st.expert_grads()  # the buffers backward() wrote (caller-supplied), not internal
    assert np.array_equal(dw1, g.dw1.cpu().numpy()) and np.array_equal(dw2, g.dw2.cpu().numpy())
    views = st.weights() if keep_views else None
    forward(st, torch.as_tensor(inp["x"]).to(torch.bfloat16).cuda())  # stats now clean
    w1, w2 = views if keep_views else st.weights()
    lr = 0.5 / float(g.dw1.abs().max())  # a step large enough to flip many ReLU signs
    w1 -= (lr * g.dw1).to(torch.bfloat16)
    w2 -= (lr * g.dw2).to(torch.bfloat16)
    if keep_views:
        st.weights_updated()
    x = torch.as_tensor(inp["x"]).to(torch.bfloat16).cuda()
    dy = torch.as_tensor(inp["dy"]).to(torch.bfloat16).cuda()
    res = forward(st, x)
    g2 = backward(st, res.saved, dy)
    torch.cuda.synchronize()
    nw1, nw2 = w1.double().cpu().numpy(), w2.double().cpu().numpy()
    assert not np.array_equal(nw1, inp["w1"])
    ref = oracle.layer_step(inp["x"], inp["wg"], nw1, nw2, inp["dy"], 1, k, 0, f, False)
    idxs, loc, _, _ = st.routing()
    assert np.array_equal(idxs, ref["idxs"]) and np.array_equal(loc, ref["locations"])
    for name, got in (("y", res.y), ("dx", g2.dx), ("dw1", g2.dw1), ("dw2", g2.dw2)):
        assert oracle.max_rel_diff(got.double().cpu().numpy(), ref[name]) < 2e-2, name
    assert st.metrics().relu_fixups > 0


def test_expert_grads_before_backward_fails(cuda):
    from paper_2206_03382_b200 import MoeError
    cfg = MoELayerConfig(global_experts=2, model_dim=64, hidden_dim=64, tokens_per_step=16)
    with pytest.raises(MoeError):
        LayerState.init(cfg, 1).expert_grads()


def test_grad_slices_single_rank(cuda):
    """reduce_scatter_grads_p1 at W = 1: the slice is the whole gradient."""
    st, res, g, ref, _ = run_case(4, 1, 1.0, 64, 256, 256, False, "f32")
    w1s, w2s = st.grad_slices()
    assert torch.equal(w1s, g.dw1) and torch.equal(w2s, g.dw2)


def test_backward_without_forward_fails(cuda):
    from paper_2206_03382_b200 import MoeError
    from paper_2206_03382_b200.layer import SavedForward
    cfg = MoELayerConfig(global_experts=2, model_dim=8, hidden_dim=8, tokens_per_step=4)
    s = LayerState.init(cfg, 1)
    with pytest.raises(MoeError):
        backward(s, SavedForward(step=0), torch.zeros(4, 8, dtype=torch.bfloat16, device="cuda"))


@pytest.mark.slow
@pytest.mark.parametrize("name,E,k,f,M,V,bpr", [("TGT", 32, 1, 1.0, 1024, 4096, False),
                                                 ("C2", 32, 1, 1.0, 768, 3072, False),
                                                 ("C3", 32, 2, 1.25, 1024, 4096, True)])
def test_layer_full_size_configs(cuda, name, E, k, f, M, V, bpr):
    """configs[1], configs[2] and the north-star TGT at full size (32K tokens): bit-exact routing
    and bf16 output/gradient parity against the fp64 oracle's per-expert GEMMs."""
    st, res, g, ref, _ = run_case(E, k, f, M, V, 32768, bpr, "bf16")
    idxs, loc, gates, cap = st.routing()
    assert np.array_equal(idxs, ref["idxs"]) and np.array_equal(loc, ref["locations"])
    assert oracle.max_rel_diff(res.y.double().cpu().numpy(), ref["y"]) < 2e-2
    assert oracle.max_rel_diff(g.dx.double().cpu().numpy(), ref["dx"]) < 2e-2
    assert oracle.max_rel_diff(g.dw1.double().cpu().numpy(), ref["dw1"]) < 2e-2
    assert oracle.max_rel_diff(g.dw2.double().cpu().numpy(), ref["dw2"]) < 2e-2


def test_fused_decode_matches_unfused(cuda, monkeypatch):
    """W = 1, k = 1: decode / encode-backward fused into the down / dgrad GEMM epilogues (TMA row
    scatter to token rows) against the unfused kernels (MOE_FUSED=0) and the oracle; drops
    included (f = 0.75), so dropped tokens' zero rows are exercised."""
    outs = {}
    for mode in ("1", "0"):
        monkeypatch.setenv("MOE_FUSED", mode)
        st, res, g, ref, _ = run_case(16, 1, 0.75, 512, 1024, 4096, False, "bf16", seed=77)
        idxs, loc, gates, cap = st.routing()
        assert np.array_equal(idxs, ref["idxs"]) and np.array_equal(loc, ref["locations"])
        assert (loc < 0).any()
        y = res.y.double().cpu().numpy()
        dx = g.dx.double().cpu().numpy()
        dropped = (ref["locations"] < 0).all(axis=1)
        assert (y[dropped] == 0).all() and (dx[dropped] == 0).all()
        for name, got in (("y", y), ("dx", dx), ("dw1", g.dw1), ("dw2", g.dw2)):
            got = got if isinstance(got, np.ndarray) else got.double().cpu().numpy()
            assert oracle.max_rel_diff(got, ref[name]) < 2e-2, (mode, name)
        outs[mode] = (res.y, g.dx, g.dw1, g.dw2)
    # same GEMMs, only the epilogue's rounding point of g * out differs
    assert torch.equal(outs["1"][1], outs["0"][1])      # dx: scatter of identical rows
    assert torch.equal(outs["1"][2], outs["0"][2]) and torch.equal(outs["1"][3], outs["0"][3])
    # y: one bf16 rounding (g * acc) vs two (acc, then g * out): within a couple of bf16 ulps
    assert oracle.max_rel_diff(outs["1"][0].double().cpu().numpy(),
                               outs["0"][0].double().cpu().numpy()) < 1e-2


def test_host_async_pipeline_matches_device_calls(cuda):
    """moe_forward_host_async / moe_backward_host_async (pipelined uploads / downloads, double-
    buffered staging) return exactly what the device-pointer calls return, step after step."""
    from paper_2206_03382_b200 import layer as L
    E, M, V, T = 8, 256, 512, 1024
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=1)
    st = LayerState.init(cfg, 21)
    xs = [(torch.rand(T, M) * 2 - 1).to(torch.bfloat16).pin_memory() for _ in range(3)]
    dys = [(torch.rand(T, M) * 2 - 1).to(torch.bfloat16).pin_memory() for _ in range(3)]
    ys = [torch.empty_like(x).pin_memory() for x in xs]
    dxs = [torch.empty_like(x).pin_memory() for x in xs]
    for i in range(3):
        L.forward_host_async(st, xs[i], ys[i])
        L.backward_host_async(st, dys[i], dxs[i])
    L.host_sync(st)
    ref = LayerState.init(cfg, 21)
    for i in range(3):
        r = forward(ref, xs[i].cuda())
        g = backward(ref, r.saved, dys[i].cuda())
        assert torch.equal(r.y.cpu(), ys[i]) and torch.equal(g.dx.cpu(), dxs[i])


@pytest.mark.parametrize("E,k,f,M,V,T,bpr,dt,cap", [
    (4, 1, 1.0, 3, 8, 8, False, "f32", "auto"),           # test_moe_layer.cpp:62-66 shape, W=1
    (16, 2, 1.25, 256, 512, 2048, True, "bf16", "fixed"),
    (32, 1, 1.0, 1024, 4096, 4096, False, "bf16", "auto"),
])
def test_layer_cosine_router(cuda, E, k, f, M, V, T, bpr, dt, cap):
    """RouterKind::Cosine inside the layer (route_probabilities, moe_layer.cpp:165-169; draws
    moe_layer.cpp:154-160): routing bit-exact, outputs / gradients at the dtype tolerance."""
    cfg = MoELayerConfig(world_size=1, global_experts=E, model_dim=M, hidden_dim=V,
                         tokens_per_step=T, top_k=k, capacity=cap, capacity_factor=f, bpr=bpr,
                         dtype=dt, router="cosine")
    inp = layer_inputs(402, 1, T, M, V, E, dt)
    st = LayerState.init(cfg, 402)
    tdt = cfg.torch_dtype
    res = forward(st, torch.as_tensor(inp["x"]).to(tdt).cuda())
    g = backward(st, res.saved, torch.as_tensor(inp["dy"]).to(tdt).cuda())
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], 1, k, kind, f,
                            bpr, cosine=(inp["cos_proj"], inp["cos_experts"], 1.0))
    idxs, loc, gates, capv = st.routing()
    assert capv == ref["capacity"]
    assert np.array_equal(idxs, ref["idxs"]) and np.array_equal(loc, ref["locations"])
    # gate values: fp64 DMMA gate (f32 / BPR layers) up to summation order; the certified
    # tensor-core gate (bf16 FIFO) carries its logit error -- ~1e-6 typical, checked at 1e-4
    certified = dt == "bf16" and not bpr and E % 8 == 0 and M % 64 == 0
    np.testing.assert_allclose(gates, ref["gates"], rtol=1e-4 if certified else 1e-12, atol=0)
    tol = 1e-5 if dt == "f32" else 2e-2
    for name, got in (("y", res.y), ("dx", g.dx), ("dw1", g.dw1), ("dw2", g.dw2)):
        assert oracle.max_rel_diff(got.double().cpu().numpy(), ref[name]) < tol, name


def test_layer_cosine_router_set_params(cuda):
    """moe_set_cosine_router (explicit RouterParams, temperature clamp) == on-device init draw."""
    E, M, V, T = 8, 64, 128, 256
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T,
                         top_k=2, router="cosine")
    inp = layer_inputs(9, 1, T, M, V, E, "bf16")
    a = LayerState.init(cfg, 9)
    b = LayerState.init(cfg, 9)
    b.set_cosine_router(inp["cos_proj"], inp["cos_experts"], 1.0)
    x = torch.as_tensor(inp["x"]).to(torch.bfloat16).cuda()
    assert torch.equal(forward(a, x).y, forward(b, x).y)
    b.set_cosine_router(inp["cos_proj"], inp["cos_experts"], 1e-9)   # clamped to 0.01
    ya = forward(b, x).y
    b.set_cosine_router(inp["cos_proj"], inp["cos_experts"], 0.01)
    assert torch.equal(ya, forward(b, x).y)
    from paper_2206_03382_b200 import MoeError
    bad = inp["cos_experts"].copy()
    bad[1] = 0.0
    with pytest.raises(MoeError):
        b.set_cosine_router(inp["cos_proj"], bad, 1.0)
