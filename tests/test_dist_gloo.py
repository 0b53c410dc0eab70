"""Multi-rank host logic on CPU (world_size 2, gloo): the flexible all-to-all plan the layer's
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
        E, dC, M, degree = 4, 5, 3, 2
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
        dist.barrier()
        dist.destroy_process_group()
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))


def test_flex_all2all_plan_world2_gloo():
    W = 2
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
