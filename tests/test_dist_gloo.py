"""Multi-rank host logic on CPU (world_size 2, 4 and 8, gloo): the flexible all-to-all plan the layer's
NCCL exchanges use (moe_a2a_plan) moves exactly the blocks of the reference flex_all2all
(collectives.cpp:123-160) for every pipeline chunk, and the per-rank token blocks / gating
blocks compose to the reference's blocked layer (moe_layer.cpp:171-244)."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _exchange(send, recv, so, ro, n, rank, W):
    ops = []
    for p in range(W):
        if p == rank:
            recv[ro[p]:ro[p] + n] = send[so[p]:so[p] + n]
            continue
        ops.append(dist.P2POp(dist.isend, send[so[p]:so[p] + n].contiguous(), p))
        ops.append(dist.P2POp(dist.irecv, recv[ro[p]:ro[p] + n], p))
    if ops:
        for r in dist.batch_isend_irecv(ops):
            r.wait()


def _worker(rank, W, port, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=W)
        import oracle
        from paper_2206_03382_b200._lib import lib
        E, dC, M, degree = 8, 5, 3, 2
        cc = -(-dC // degree)
        dE = E // W
        rs = np.random.RandomState(100)
        inputs = rs.uniform(-1, 1, (W, E, dC, M))          # every rank's (E, dC, M) slab
        mine = inputs[rank]
        chunks = oracle.partition_capacity(mine, degree)    # (degree, E, cc, M): send layout
        send = torch.from_numpy(chunks.copy()).reshape(-1)
        recv = torch.zeros(degree * W * dE * cc * M, dtype=torch.float64)
        so = (C.c_int64 * W)()
        ro = (C.c_int64 * W)()
        n = C.c_int64()
        for i in range(degree):
            assert lib().moe_a2a_plan(W, E, cc, M, i, 0, so, ro, C.byref(n)) == 0
            _exchange(send, recv, list(so), list(ro), n.value, rank, W)
        got = recv.numpy().reshape(degree, W, dE, cc, M)
        # reference: flex dispatch of each chunk, then expert e's rows (r, c) of chunk i
        part = np.stack([oracle.partition_capacity(inputs[r], degree) for r in range(W)])
        for i in range(degree):
            want = oracle.flex_dispatch(part[:, i], W)[rank]  # (dE, W*cc, M)
            for r in range(W):
                for e in range(dE):
                    assert np.array_equal(got[i, r, e], want[e, r * cc:(r + 1) * cc])
        # combine is the exact inverse
        back = torch.zeros_like(send)
        for i in range(degree):
            assert lib().moe_a2a_plan(W, E, cc, M, i, 1, so, ro, C.byref(n)) == 0
            _exchange(recv, back, list(so), list(ro), n.value, rank, W)
        assert np.array_equal(back.numpy(), chunks.reshape(-1))
        # per-rank token blocks: gating my block alone == the reference's blocked gating rows
        T, Mx, Ex, k = 6, 4, 4, 2
        x = rs.uniform(-1, 1, (W * T, Mx))
        wg = rs.uniform(-1, 1, (Mx, Ex))
        probs = oracle.gate_linear(x, wg)
        gi, gg, gl, cap = oracle.run_gating_blocked(probs, W, k, 0, 1.0, True)
        li, lg, ll, lcap = oracle.run_gating_blocked(probs[rank * T:(rank + 1) * T], 1, k, 0, 1.0, True)
        assert cap == lcap
        assert np.array_equal(li, gi[rank * T:(rank + 1) * T])
        assert np.array_equal(ll, gl[rank * T:(rank + 1) * T])
        # Auto capacity across ranks (gating.cpp:141-147): per-rank demand, all-reduce MAX (the
        # layer's ncclAllReduce), resolve, assign my block == the reference's blocked gating
        for kind, fac in ((1, 1.0), (2, 1.25), (2, 0.5)):
            gi, gg, gl, cap = oracle.run_gating_blocked(probs, W, k, kind, fac, True)
            dem = torch.from_numpy(np.bincount(li.ravel(), minlength=Ex).astype(np.int64))
            dist.all_reduce(dem, op=dist.ReduceOp.MAX)
            lcap = oracle.resolve_capacity(kind, fac, dem.numpy(), Ex, k, T)
            assert lcap == cap
            assert np.array_equal(oracle.assign_locations(li, lg, lcap, True), gl[rank * T:(rank + 1) * T])
        # Alg. 1 consensus: each rank measures its own seconds, the layer all-reduces the max
        # before recording, so every rank's memo explores and exploits the same strategies
        memo = C.c_void_p()
        assert lib().moe_memo_create(C.c_double(0.5), C.byref(memo)) == 0
        picks = []
        s = C.c_int32()
        for step in range(14):
            f = (1.0, 1.2, 2.0)[step % 3]
            assert lib().moe_memo_get_strategy(memo, C.c_double(f), C.byref(s)) == 0
            picks.append(s.value)
            t = torch.tensor([float(rs.uniform(1, 2)) * (1 + rank) + s.value * 0.01])
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            assert lib().moe_memo_optimize_strategy(memo, C.c_double(f), s, C.c_double(t.item())) == 0
        lib().moe_memo_destroy(memo)
        allp = [None] * W
        dist.all_gather_object(allp, picks)
        assert all(p == picks for p in allp)
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


@pytest.mark.parametrize("W", [2, 4, 8])
def test_flex_all2all_plan_gloo(W):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, W, port, q)) for r in range(W)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(W))
    for p in procs:
        p.join(timeout=60)
    for r in range(W):
        assert results[r] == "ok", results[r]
