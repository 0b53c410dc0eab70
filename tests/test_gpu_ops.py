"""GPU sub-operator parity against the fp64 oracle and the reference KATs.

Routing (idxs, locations, drop mask) must be bit-exact; gates/probs to 1e-12 relative; encode
and dispatch layouts byte-exact; decode / FFN within the dtype tolerance (max_rel_diff as in
tensor.cpp:52-55).
"""
import json
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2206_03382_b200 import ops, rng
from tests.helpers import probs_to_inputs, row_probs

pytestmark = pytest.mark.gpu

KATS = json.loads((Path(__file__).parent / "golden" / "reference_kats.json").read_text())


def t(a, dtype, dev):
    return torch.as_tensor(np.ascontiguousarray(a), device=dev).to(dtype).contiguous()


def gpu_gating(x, wg, blocks, k, cap="fixed", factor=1.0, bpr=False, dtype=torch.float32, probs=False):
    dev = torch.device("cuda:0")
    idxs, gates, loc, c, drops, p = ops.gating(t(x, dtype, dev), t(wg, torch.float64, dev), blocks, k,
                                               cap, factor, bpr, want_probs=probs)
    torch.cuda.synchronize()
    out = dict(idxs=idxs.cpu().numpy(), gates=gates.cpu().numpy(), loc=loc.cpu().numpy(), cap=c,
               drops=drops)
    if probs:
        out["probs"] = p.cpu().numpy()
    return out


# ---------------------------------------------------------------- KATs on the device
def test_kat_softmax(cuda):
    for case in KATS["softmax"]:
        g = gpu_gating(np.array(case["x"]), np.array(case["wg"]), 1, 1, probs=True)
        np.testing.assert_allclose(g["probs"], np.array(case["probs"]), rtol=0, atol=1e-15)


def test_kat_topk_tie_break(cuda):
    for case in KATS["topk"]:
        x, wg = probs_to_inputs(case["probs"])
        g = gpu_gating(x, wg, 1, case["k"], cap="auto")
        assert g["idxs"].tolist() == case["idxs"], case["src"]
        assert abs(g["gates"][0, 0] - case["gate00"]) < 1e-15


@pytest.mark.parametrize("case", KATS["assign_locations"], ids=lambda c: c["src"])
def test_kat_assign_locations(cuda, case):
    E = 8
    probs = np.stack([row_probs(i, g, E) for i, g in zip(case["idxs"], case["gates"])])
    x, wg = probs_to_inputs(probs)
    T = len(case["idxs"])
    # fixed capacity cap = ceil(f*T/E): choose f so the resolved capacity equals the KAT's
    f = case["cap"] * E / T
    g = gpu_gating(x, wg, 1, 1, "fixed", f, bool(case["bpr"]))
    assert g["cap"] == case["cap"]
    assert g["idxs"][:, 0].tolist() == case["idxs"]
    assert g["loc"][:, 0].tolist() == case["locations"], case["src"]


@pytest.mark.parametrize("case", KATS["run_gating"], ids=lambda c: c["src"])
def test_kat_run_gating(cuda, case):
    x, wg = probs_to_inputs(case["probs"])
    cap = {0: "fixed", 1: "auto", 2: "bounded"}[case["kind"]]
    g = gpu_gating(x, wg, case["blocks"], case["k"], cap, case["factor"] or 1.0)
    assert g["cap"] == case["cap"]
    if "drops" in case:
        assert g["drops"] == case["drops"]
    if "locations" in case:
        assert g["loc"][:, 0].tolist() == case["locations"]


def test_kat_encode(cuda):
    dev = torch.device("cuda:0")
    for case in KATS["encode"]:
        x = t(case["x"], torch.float32, dev)
        idxs = t(np.array(case["idxs"]).reshape(-1, 1), torch.int32, dev)
        loc = t(np.array(case["locations"]).reshape(-1, 1), torch.int32, dev)
        z = ops.encode(x, 1, case["E"], 1, case["cap"], 1, idxs, loc)
        assert z[0, 0].cpu().tolist() == case["z"]


def test_kat_expert_ffn(cuda):
    dev = torch.device("cuda:0")
    for case in KATS["expert_ffn"]:
        y = ops.expert_ffn(t(case["x"], torch.float32, dev), t(case["w1"], torch.float32, dev),
                           t(case["w2"], torch.float32, dev))
        assert y.cpu().tolist() == case["y"], case["src"]


# ---------------------------------------------------------------- randomized routing parity
GATING_CASES = [
    # blocks, T, M, E, k, cap kind, factor, bpr, dtype
    (1, 4096, 512, 8, 1, "fixed", 1.0, False, "f32"),      # C1 routing
    (2, 1000, 64, 16, 2, "fixed", 1.25, True, "bf16"),
    (4, 333, 48, 24, 2, "fixed", 0.5, True, "bf16"),       # heavy drops, ragged T
    (3, 200, 40, 64, 4, "auto", 1.0, False, "bf16"),
    (2, 512, 96, 64, 2, "bounded", 1.0, True, "f32"),
    (1, 32768, 1024, 32, 1, "fixed", 1.0, False, "bf16"),  # TGT routing
    (1, 32768, 1024, 32, 2, "fixed", 1.25, True, "bf16"),  # C3 routing (top-2 + BPR)
    (1, 7, 5, 3, 3, "fixed", 1.0, True, "f32"),           # k = E, tiny, ragged
    (2, 4096, 32, 2, 2, "fixed", 0.5, True, "f32"),       # BPR lists of exactly 4096 (sort width)
    (1, 20000, 32, 2, 1, "fixed", 0.8, True, "f32"),      # BPR lists > 8192: pairwise fallback
]


@pytest.mark.parametrize("case", GATING_CASES, ids=str)
def test_gating_bit_exact(cuda, case):
    blocks, T, M, E, k, cap, f, bpr, dt = case
    seed = 402 + T + E
    x = rng.round_dtype(rng.uniform(seed, 0, blocks * T * M).reshape(blocks * T, M), dt)
    wg = rng.uniform(seed, blocks * T * M, M * E).reshape(M, E)
    g = gpu_gating(x, wg, blocks, k, cap, f, bpr, torch.bfloat16 if dt == "bf16" else torch.float32)
    probs = oracle.gate_linear(x, wg)
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    oi, og, ol, ocap = oracle.run_gating_blocked(probs, blocks, k, kind, f, bpr)
    assert g["cap"] == ocap
    assert np.array_equal(g["idxs"], oi), "gate indices differ"
    assert np.array_equal(g["loc"], ol), "capacity locations differ"
    assert g["drops"] == int((ol < 0).sum())
    np.testing.assert_allclose(g["gates"], og, rtol=1e-12, atol=0)


# ---------------------------------------------------------------- dispatch parity
DISPATCH_CASES = [
    # blocks, T, M, E, k, f, bpr, degree, dtype
    (1, 300, 64, 8, 1, 1.0, False, 1, torch.float32),
    (2, 257, 40, 6, 2, 0.7, True, 4, torch.float32),      # non-vector M, drops, chunks
    (1, 2048, 1024, 32, 1, 1.0, False, 2, torch.bfloat16),
    (3, 100, 128, 8, 2, 1.5, False, 8, torch.bfloat16),   # degree > ... padded tail
]


@pytest.mark.parametrize("case", DISPATCH_CASES, ids=str)
def test_dispatch_parity(cuda, case):
    blocks, T, M, E, k, f, bpr, degree, tdt = case
    dev = torch.device("cuda:0")
    dts = "bf16" if tdt == torch.bfloat16 else "f32"
    seed = 43 + T
    x = rng.round_dtype(rng.uniform(seed, 0, blocks * T * M).reshape(blocks * T, M), dts)
    wg = rng.uniform(seed, 10 ** 7, M * E).reshape(M, E)
    xd = t(x, tdt, dev)
    idxs, gates, loc, cap, _, _ = ops.gating(xd, t(wg, torch.float64, dev), blocks, k, "fixed", f, bpr)
    oi, og, ol = idxs.cpu().numpy(), gates.cpu().numpy(), loc.cpu().numpy()
    # encode: byte-exact vs oracle encode + partition_capacity
    z = ops.encode(xd, blocks, E, k, cap, degree, idxs, loc)
    oz = oracle.encode(x, blocks, E, k, cap, oi, ol)
    want = np.stack([oracle.partition_capacity(oz[b], degree) for b in range(blocks)])
    assert np.array_equal(z.double().cpu().numpy(), want)
    if blocks == 1:
        assert np.array_equal(oz[0], oracle.encode_dense(x, E, k, cap, oi, ol))
    # decode of a random expert output
    ze = rng.round_dtype(rng.uniform(seed + 1, 0, z.numel()).reshape(z.shape), dts)
    y = ops.decode(t(ze, tdt, dev), blocks, T, k, cap, idxs, loc, gates)
    merged = np.stack([oracle.merge_chunks(ze[b], cap) for b in range(blocks)])
    oy = oracle.decode(merged, blocks, T, k, oi, ol, og)
    tol = 1e-6 if tdt == torch.float32 else 1e-2
    assert oracle.max_rel_diff(y.double().cpu().numpy(), oy) < tol
    dropped = (ol < 0).all(axis=1)
    assert (y.cpu()[torch.from_numpy(dropped)] == 0).all()
    # decode backward (dz and d_gates) and encode backward
    dy = rng.round_dtype(rng.uniform(seed + 2, 0, blocks * T * M).reshape(blocks * T, M), dts)
    dz, dg = ops.decode_backward(t(dy, tdt, dev), t(ze, tdt, dev), blocks, E, k, cap, degree,
                                 idxs, loc, gates, want_dgates=True)
    odz, odg = oracle.decode_backward(dy, merged, blocks, E, k, cap, oi, ol, og)
    want = np.stack([oracle.partition_capacity(odz[b], degree) for b in range(blocks)])
    assert oracle.max_rel_diff(dz.double().cpu().numpy(), want) < tol
    assert oracle.max_rel_diff(dg.cpu().numpy(), odg) < 1e-5
    dx = ops.encode_backward(t(ze, tdt, dev), blocks, T, k, cap, idxs, loc)
    odx = oracle.encode_backward(merged, blocks, T, k, oi, ol)
    assert oracle.max_rel_diff(dx.double().cpu().numpy(), odx) < tol


# ---------------------------------------------------------------- expert FFN parity
@pytest.mark.parametrize("n,rows,M,V,dt", [(2, 96, 32, 48, "f32"), (3, 256, 256, 512, "bf16"),
                                           (2, 200, 512, 1024, "bf16")])
def test_expert_ffn_parity(cuda, n, rows, M, V, dt):
    dev = torch.device("cuda:0")
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    seed = 7 + rows
    x = rng.round_dtype(rng.uniform(seed, 0, n * rows * M).reshape(n, rows, M), dt)
    w1 = rng.round_dtype(rng.uniform(seed, 10 ** 8, n * M * V, -0.5, 0.5).reshape(n, M, V), dt)
    w2 = rng.round_dtype(rng.uniform(seed, 2 * 10 ** 8, n * V * M, -0.5, 0.5).reshape(n, V, M), dt)
    dy = rng.round_dtype(rng.uniform(seed, 3 * 10 ** 8, n * rows * M).reshape(n, rows, M), dt)
    y = ops.expert_ffn(t(x, tdt, dev), t(w1, tdt, dev), t(w2, tdt, dev))
    oy = oracle.expert_ffn(x, w1, w2)
    tol = 1e-5 if dt == "f32" else 2e-2
    assert oracle.max_rel_diff(y.double().cpu().numpy(), oy) < tol
    dx, dw1, dw2 = ops.expert_ffn_backward(t(x, tdt, dev), t(w1, tdt, dev), t(w2, tdt, dev),
                                           t(dy, tdt, dev))
    odx, odw1, odw2 = oracle.expert_ffn_backward(x, w1, w2, dy)
    assert oracle.max_rel_diff(dx.double().cpu().numpy(), odx) < tol
    assert oracle.max_rel_diff(dw1.double().cpu().numpy(), odw1) < tol
    assert oracle.max_rel_diff(dw2.double().cpu().numpy(), odw2) < tol


def test_fill_uniform_matches_host_stream(cuda):
    dev = torch.device("cuda:0")
    out = torch.empty(100000, dtype=torch.float64, device=dev)
    ops.fill_uniform(out, 402, 12345, -0.5, 0.5)
    assert np.array_equal(out.cpu().numpy(), rng.uniform(402, 12345, 100000, -0.5, 0.5))
    ob = torch.empty(100000, dtype=torch.bfloat16, device=dev)
    ops.fill_uniform(ob, 402, 12345, -0.5, 0.5)
    assert np.array_equal(ob.double().cpu().numpy(),
                          rng.round_bf16(rng.uniform(402, 12345, 100000, -0.5, 0.5)))


# ---------------------------------------------------------------- cosine router parity
COSINE_CASES = [
    # blocks, T, M, E, k, cap kind, factor, bpr, dtype, temperature
    (1, 2048, 256, 8, 1, "fixed", 1.0, False, "bf16", 1.0),
    (2, 1000, 64, 32, 2, "auto", 1.0, True, "bf16", 0.07),
    (3, 333, 40, 64, 2, "fixed", 0.5, True, "f32", 1e-9),   # temperature clamped to 0.01
    (1, 32768, 1024, 32, 1, "fixed", 1.0, False, "bf16", 1.0),  # TGT shape
]


@pytest.mark.parametrize("case", COSINE_CASES, ids=str)
def test_cosine_gating_matches_oracle(cuda, case):
    """gate_cosine (gating.cpp:37-56) + run_gating_blocked on the GPU (fp64 DMMA projection and
    cosine logits) against the oracle: routing bit-exact, gates to 1e-12."""
    from paper_2206_03382_b200 import ops
    blocks, T, M, E, k, cap, f, bpr, dt, tau = case
    seed = 77 + T + E
    x = rng.round_dtype(rng.uniform(seed, 0, blocks * T * M).reshape(blocks * T, M), dt)
    proj = rng.uniform(seed, blocks * T * M, M * 256).reshape(M, 256)
    experts = rng.uniform(seed, blocks * T * M + M * 256, E * 256).reshape(E, 256)
    tdt = torch.bfloat16 if dt == "bf16" else torch.float32
    xi = torch.as_tensor(x).to(tdt).cuda()
    idxs, gates, loc, gcap, drops, probs = ops.gating_cosine(
        xi, torch.as_tensor(proj).cuda(), torch.as_tensor(experts).cuda(), blocks, k, tau, cap, f,
        bpr, want_probs=True)
    oprobs = oracle.gate_cosine(x, proj, experts, tau)
    np.testing.assert_allclose(probs.cpu().numpy(), oprobs, rtol=1e-11, atol=1e-300)
    kind = {"fixed": 0, "auto": 1, "bounded": 2}[cap]
    oi, og, ol, ocap = oracle.run_gating_blocked(oprobs, blocks, k, kind, f, bpr)
    assert gcap == ocap
    assert np.array_equal(idxs.cpu().numpy(), oi) and np.array_equal(loc.cpu().numpy(), ol)
    assert drops == int((ol < 0).sum())
    np.testing.assert_allclose(gates.cpu().numpy(), og, rtol=1e-12, atol=0)


def test_cosine_gating_rejects_zero_norms(cuda):
    """A zero-norm expert row or projected token raises invalid_argument (gating.cpp:46-49)."""
    from paper_2206_03382_b200 import ops, MoeError
    x = torch.rand(128, 64, device="cuda").to(torch.bfloat16)
    proj = torch.rand(64, 256, device="cuda", dtype=torch.float64) - 0.5
    experts = torch.rand(8, 256, device="cuda", dtype=torch.float64) - 0.5
    experts[3] = 0.0
    with pytest.raises(MoeError):
        ops.gating_cosine(x, proj, experts, 1, 1)
    experts[3] = 1.0
    x[5] = 0.0
    with pytest.raises(MoeError):
        ops.gating_cosine(x, proj, experts, 1, 1)


@pytest.mark.parametrize("n,M,V", [(2, 1024, 4096), (3, 64, 192), (1, 40, 72)])
def test_weight_stats_matches_torch(cuda, n, M, V):
    """The ReLU certificate's weight statistics (one-pass kernel for M, V multiples of 64; the
    generic kernels otherwise): W1^T bit-exact, column norms >= the fp64 norm and within 2e-4."""
    from paper_2206_03382_b200 import ops
    w1 = (torch.rand(n, M, V, device="cuda", dtype=torch.float64) - 0.5).to(torch.bfloat16)
    colnorm, blk, w1t = ops.weight_stats(w1)
    torch.cuda.synchronize()
    assert torch.equal(w1t, w1.transpose(1, 2).contiguous())
    ref = w1.double().pow(2).sum(dim=1).sqrt()
    cn = colnorm.double()
    assert (cn >= ref * (1 - 1e-7)).all() and ((cn - ref) / ref).abs().max() < 2e-4
    if V % 64 == 0:
        assert torch.equal(blk, colnorm.view(n, V // 64, 64).amax(dim=2))
