"""Full-shape expert-parallel parity for BASELINE configs[3] (C4) on W GPUs, plus strategy
invariance. Launch one rank per GPU:

    torchrun --nproc-per-node W tools/mp_parity_c4.py [--tokens 65536 --M 1024 --V 4096 --epr 8]

C4 per rank: E = 8W experts (8 per GPU), k = 1, f = 1.0, M = 1024, V = 4096, 65 536 tokens per
rank, bf16, seed 402 (LayerState::init draw order, x / dy drawn after it; test_moe_layer.cpp:70-73).

Every (transport, degree) run -- peer (copy-engine dispatch + NVLink-fused combine), peer-fd
(dispatch fused into the encode / decode-backward kernels as NVLink stores) and NCCL, at
pipelining degrees 1 / 2 / 4 / 8, and Alg. 1 adaptive -- is checked for:
* strategy invariance (test_moe_layer.cpp:82-100): routing, y and dx bit-identical to the
  degree-1 peer run; dW1 / dW2 within 1e-5 (the wgrad K-loop visits the capacity chunks in a
  different grouping);
and the degree-1 peer run against the fp64 oracle (SURVEY §8c "resulting parity design"):
* routing (expert ids, slots, drops, capacity) bit-exact over all W*T tokens, gate values
  within the certified gate's bound (2^-18 |x_t| max|Wg_e|, relative): each rank's block against orc_gate_linear +
  orc_run_gating_blocked on that block (Fixed capacity gates blocks independently,
  gating.cpp:134-162); a failure on any rank fails all;
* y and dx on a sampled token subset (incl. dropped tokens) through the frozen-plan oracle
  (moe_layer.cpp:321-335 forward, :246-319 backward per token), 2e-2 (north_star bf16);
* dW1 columns / dW2 rows of sampled hidden units of every local expert, from the expert's rows
  gathered from all W source blocks (parallelism.cpp:123-147), 2e-2.
Rank 0 prints one PASS/FAIL line per check; exit code 0 iff all pass on every rank.
"""
import argparse
import os
import sys
import time

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (the checker; test infrastructure)
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward, rng  # noqa: E402

SEED = 402
TOL = 2e-2
DW_INVARIANCE_TOL = 1e-5


def draws(offset, n, lo=-1.0, hi=1.0):
    return oracle.fill_uniform(SEED, offset, n, lo, hi)


def expert_weights(off, M, V, experts):
    """w1 (n, M, V), w2 (n, V, M) of the given global experts, bf16-rounded fp64."""
    w1 = np.empty((len(experts), M, V))
    w2 = np.empty((len(experts), V, M))
    for i, e in enumerate(experts):
        o = off["experts"] + e * off["expert_stride"]
        w1[i] = rng.round_bf16(draws(o, M * V, -0.5, 0.5)).reshape(M, V)
        w2[i] = rng.round_bf16(draws(o + M * V, V * M, -0.5, 0.5)).reshape(V, M)
    return w1, w2


def say(rank, *a):
    if rank == 0:
        print(*a, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", type=int, default=65536)
    ap.add_argument("--M", type=int, default=1024)
    ap.add_argument("--V", type=int, default=4096)
    ap.add_argument("--epr", type=int, default=8, help="experts per rank")
    ap.add_argument("--samples", type=int, default=48)
    ap.add_argument("--cols", type=int, default=6, help="sampled hidden units per local expert")
    ap.add_argument("--degrees", default="1,2,4,8")
    a = ap.parse_args()
    rank, W, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    oracle.set_num_threads(max(1, (os.cpu_count() or W) // W))
    T, M, V, E, k, f = a.tokens, a.M, a.V, a.epr * W, 1, 1.0
    off = rng.draw_offsets(M, E, V, W, T)
    t0 = time.time()
    x_np = rng.round_bf16(draws(off["x"] + rank * T * M, T * M)).reshape(T, M)
    dy_np = rng.round_bf16(draws(off["dy"] + rank * T * M, T * M)).reshape(T, M)
    wg = draws(off["wg"], M * E).reshape(M, E)
    x = torch.from_numpy(x_np).to(torch.bfloat16).to(dev)
    dy = torch.from_numpy(dy_np).to(torch.bfloat16).to(dev)
    say(rank, f"C4 parity: W={W} E={E} k={k} f={f} M={M} V={V} T/rank={T} (inputs {time.time() - t0:.1f}s)")

    # ---- every strategy on the same inputs
    runs = [("peer", d, False) for d in map(int, a.degrees.split(","))]
    runs += [("nccl", d, False) for d in (1, max(map(int, a.degrees.split(","))))]
    runs += [("peer-fd", d, False) for d in (1, 4)]  # dispatch fused into encode (NVLink stores)
    runs += [("peer-parts", 1, False)]  # chunk 0 in 2-tile row parts (MOE_PARTS) instead of thirds
    runs += [("peer", 1, True)]
    base = None
    all_ok = True

    def agree(flag):
        t = torch.tensor([0.0 if flag else 1.0], device=dev)
        dist.all_reduce(t)
        return t.item() == 0

    for backend, degree, adaptive in runs:
        fd = backend == "peer-fd"
        if fd:
            os.environ["MOE_DISPATCH"] = "fused"
        if backend == "peer-parts":  # capacity 8192 / W rows = 32 / W tiles of 256
            os.environ["MOE_PARTS"] = ",".join(["2"] * (16 // W))
        cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=E, model_dim=M,
                             hidden_dim=V, tokens_per_step=T, top_k=k, capacity_factor=f,
                             dtype="bf16", degree=degree, adaptive=adaptive,
                             a2a_backend="peer" if backend.startswith("peer") else backend)
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        st = LayerState.init(cfg, SEED, rank=rank, device=local, nccl_id=obj[0])
        os.environ.pop("MOE_DISPATCH", None)
        steps = 20 if adaptive else 2
        for _ in range(steps):
            res = forward(st, x)
            g = backward(st, res.saved, dy)
        torch.cuda.synchronize()
        os.environ.pop("MOE_PARTS", None)
        idxs, loc, gates, cap = st.routing()
        m = st.metrics()
        out = dict(y=res.y.clone(), dx=g.dx.clone(), dw1=g.dw1.clone(), dw2=g.dw2.clone(),
                   idxs=idxs, loc=loc, gates=gates, cap=cap)
        name = f"{backend} degree={m.degree}{' (adaptive)' if adaptive else ''}"
        if base is None:
            base = out
            ok = agree(True)
        else:
            e = dict(routing=int(not (np.array_equal(idxs, base["idxs"]) and np.array_equal(loc, base["loc"])
                                      and np.array_equal(gates, base["gates"]))),
                     y_bits=int(not torch.equal(out["y"], base["y"])),
                     dx_bits=int(not torch.equal(out["dx"], base["dx"])),
                     dw1=oracle.max_rel_diff(out["dw1"].double().cpu().numpy(), base["dw1"].double().cpu().numpy()),
                     dw2=oracle.max_rel_diff(out["dw2"].double().cpu().numpy(), base["dw2"].double().cpu().numpy()))
            ok = agree(e["routing"] == 0 and e["y_bits"] == 0 and e["dx_bits"] == 0
                       and e["dw1"] < DW_INVARIANCE_TOL and e["dw2"] < DW_INVARIANCE_TOL)
            say(rank, "PASS" if ok else "FAIL", f"invariance {name} vs peer degree=1:", e,
                f"ms/step={m.seconds * 1e3:.3f}")
        all_ok &= ok
        st.close()
        del res, g

    # ---- degree-1 peer run against the oracle
    t0 = time.time()
    probs = oracle.gate_linear(x_np, wg)
    r_idx, r_gates, r_loc, r_cap = oracle.run_gating_blocked(probs, 1, k, 0, f, False)
    del probs
    routing_ok = (np.array_equal(base["idxs"].reshape(T, k), r_idx) and
                  np.array_equal(base["loc"].reshape(T, k), r_loc) and
                  base["cap"] == r_cap)
    # gate values: the certified tensor-core gate's logit error (tests/test_gpu_gate_tc.py bound)
    xn = np.linalg.norm(x_np, axis=1)[:, None]
    gbound = 2.0 ** -18 * xn * np.linalg.norm(wg, axis=0).max()
    with np.errstate(divide="ignore", invalid="ignore"):
        grel = np.where(base["gates"].reshape(T, k) == r_gates, 0.0,
                        np.abs(base["gates"].reshape(T, k) - r_gates) / np.abs(r_gates))
    routing_ok = routing_ok and bool((grel <= np.maximum(gbound, 1e-12)).all())
    ok = agree(routing_ok)
    all_ok &= ok
    drops = int((r_loc < 0).all(axis=1).sum())
    say(rank, "PASS" if ok else "FAIL", f"routing bit-exact on all {W}x{T} tokens (capacity {r_cap}, "
        f"rank-0 drops {drops}, oracle gating {time.time() - t0:.1f}s)")

    # sampled tokens: random kept ones plus dropped ones
    gen = np.random.default_rng(1000 + rank)
    dropped = np.nonzero((r_loc < 0).all(axis=1))[0]
    sel = np.unique(np.concatenate([gen.choice(T, a.samples, replace=False),
                                    dropped[:8], [0, T - 1]])).astype(np.int64)
    experts = sorted(set(int(e) for e in r_idx[sel].ravel()))
    w1s, w2s = expert_weights(off, M, V, experts)
    remap = {e: i for i, e in enumerate(experts)}
    sidx = np.vectorize(remap.get)(r_idx[sel]).astype(np.int64)
    t0 = time.time()
    y_ref = oracle.frozen_plan_forward(x_np[sel], k, sidx, r_loc[sel], r_gates[sel], w1s, w2s)
    dx_ref = oracle.frozen_plan_backward_rows(x_np[sel], dy_np[sel], k, sidx, r_loc[sel], r_gates[sel], w1s, w2s)
    sel_t = torch.from_numpy(sel).to(dev)
    ey = oracle.max_rel_diff(base["y"].index_select(0, sel_t).double().cpu().numpy(), y_ref)
    edx = oracle.max_rel_diff(base["dx"].index_select(0, sel_t).double().cpu().numpy(), dx_ref)
    zero_drop = bool((base["y"].index_select(0, torch.from_numpy(dropped).to(dev)) == 0).all()) if len(dropped) else True
    ok = agree(ey < TOL and edx < TOL and zero_drop)
    all_ok &= ok
    say(rank, "PASS" if ok else "FAIL", f"y / dx on {len(sel)} sampled tokens per rank "
        f"(rank 0: y {ey:.2e}, dx {edx:.2e}, dropped rows zero: {zero_drop}; {time.time() - t0:.1f}s)")

    # dW of sampled hidden units: every local expert's rows from all W source blocks
    t0 = time.time()
    xs_all = [torch.empty_like(x) for _ in range(W)]
    dys_all = [torch.empty_like(dy) for _ in range(W)]
    dist.all_gather(xs_all, x)
    dist.all_gather(dys_all, dy)
    rt = [torch.empty(T * k, dtype=torch.int32, device=dev) for _ in range(W)]
    lt = [torch.empty(T * k, dtype=torch.int32, device=dev) for _ in range(W)]
    gt = [torch.empty(T * k, dtype=torch.float64, device=dev) for _ in range(W)]
    dist.all_gather(rt, torch.from_numpy(base["idxs"]).to(dev))
    dist.all_gather(lt, torch.from_numpy(base["loc"]).to(dev))
    dist.all_gather(gt, torch.from_numpy(base["gates"]).to(dev))
    idx_all = torch.cat(rt).view(W * T, k)  # routing verified bit-exact on every rank above
    loc_all = torch.cat(lt).view(W * T, k)
    g_all = torch.cat(gt).view(W * T, k)
    x_all = torch.cat(xs_all)
    dy_all = torch.cat(dys_all)
    local_e = list(range(rank * a.epr, (rank + 1) * a.epr))
    w1l, w2l = expert_weights(off, M, V, local_e)
    worst1 = worst2 = 0.0
    for i, e in enumerate(local_e):
        t_, j_ = torch.nonzero((idx_all == e) & (loc_all >= 0), as_tuple=True)
        X = x_all.index_select(0, t_).double().cpu().numpy()
        dZ = (g_all[t_, j_][:, None] * dy_all.index_select(0, t_).double()).cpu().numpy()
        cols = np.sort(gen.choice(V, a.cols, replace=False)).astype(np.int64)
        d1, d2 = oracle.expert_backward_columns(X, dZ, w1l[i], w2l[i], cols)
        g1 = base["dw1"][i][:, torch.from_numpy(cols).to(dev)].double().cpu().numpy()
        g2 = base["dw2"][i][torch.from_numpy(cols).to(dev), :].double().cpu().numpy()
        worst1 = max(worst1, oracle.max_rel_diff(g1, d1))
        worst2 = max(worst2, oracle.max_rel_diff(g2, d2))
    ok = agree(worst1 < TOL and worst2 < TOL)
    all_ok &= ok
    say(rank, "PASS" if ok else "FAIL", f"dW1 columns / dW2 rows, {a.cols} hidden units x {a.epr} local "
        f"experts per rank (rank 0: dw1 {worst1:.2e}, dw2 {worst2:.2e}; {time.time() - t0:.1f}s)")
    say(rank, "ALL PASS" if all_ok else "SOME FAILED")
    dist.destroy_process_group()
    sys.exit(0 if all_ok else 1)


if __name__ == "__main__":
    main()
