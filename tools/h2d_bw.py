"""Host<->device copy bandwidth on the box (pinned buffers): one stream vs two streams per
direction, each direction alone and both at once -- the ceiling of the e2e (host-buffer) path."""
import torch


def run(n_mb=64, reps=20):
    dev = torch.device("cuda", 0)
    n = n_mb << 20
    h = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
    o = [torch.empty(n, dtype=torch.uint8).pin_memory() for _ in range(2)]
    d = [torch.empty(n, dtype=torch.uint8, device=dev) for _ in range(4)]
    ss = [torch.cuda.Stream(dev) for _ in range(4)]

    def timed(fn):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss:
            s.wait_event(e0)
        fn()
        for s in ss:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        e1.synchronize()
        return e0.elapsed_time(e1) * 1e-3

    def h2d(streams):
        for r in range(reps):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    d[i].copy_(h[i % 2], non_blocking=True)

    def d2h(streams):
        for r in range(reps):
            for i, s in enumerate(streams):
                with torch.cuda.stream(s):
                    o[i % 2].copy_(d[2 + i], non_blocking=True)

    for name, fn, nbytes in [
        ("h2d 1 stream", lambda: h2d(ss[:1]), reps * n),
        ("h2d 2 streams", lambda: h2d(ss[:2]), 2 * reps * n),
        ("d2h 1 stream", lambda: d2h(ss[2:3]), reps * n),
        ("d2h 2 streams", lambda: d2h(ss[2:4]), 2 * reps * n),
        ("h2d+d2h 1+1", lambda: (h2d(ss[:1]), d2h(ss[2:3])), 2 * reps * n),
        ("h2d+d2h 2+2", lambda: (h2d(ss[:2]), d2h(ss[2:4])), 4 * reps * n),
    ]:
        fn()
        t = timed(fn)
        print(f"{name:16s} {nbytes / t / 1e9:7.1f} GB/s total")


if __name__ == "__main__" and "RANK" not in __import__("os").environ:
    run()


def run_multi(n_mb=64, reps=20):
    """Every visible GPU copying both directions at once (one process): the box's aggregate
    host<->device bandwidth, which bounds the e2e path at N > 1."""
    import time
    ng = torch.cuda.device_count()
    n = n_mb << 20
    bufs = []
    for g in range(ng):
        dev = torch.device("cuda", g)
        bufs.append(dict(h=torch.empty(n, dtype=torch.uint8).pin_memory(),
                         o=torch.empty(n, dtype=torch.uint8).pin_memory(),
                         d=torch.empty(n, dtype=torch.uint8, device=dev),
                         e=torch.empty(n, dtype=torch.uint8, device=dev),
                         s1=torch.cuda.Stream(dev), s2=torch.cuda.Stream(dev)))

    for dirs in (("h2d",), ("d2h",), ("h2d", "d2h")):
        for use in range(1, ng + 1):
            def go():
                for _ in range(reps):
                    for b in bufs[:use]:
                        if "h2d" in dirs:
                            with torch.cuda.stream(b["s1"]):
                                b["d"].copy_(b["h"], non_blocking=True)
                        if "d2h" in dirs:
                            with torch.cuda.stream(b["s2"]):
                                b["o"].copy_(b["e"], non_blocking=True)
            go()
            for g in range(ng):
                torch.cuda.synchronize(g)
            t0 = time.perf_counter()
            go()
            for g in range(ng):
                torch.cuda.synchronize(g)
            el = time.perf_counter() - t0
            tot = reps * n * len(dirs) * use
            print(f"{'+'.join(dirs):8s} on {use} GPU(s): {tot / el / 1e9:7.1f} GB/s aggregate")


if __name__ == "__main__" and torch.cuda.device_count() > 1 and "RANK" not in __import__("os").environ:
    run_multi()


def run_ranks(n_mb=128, reps=10):
    """torchrun: one process per GPU, both directions at once after a barrier -- the e2e
    path's layout (separate processes, separately pinned buffers)."""
    import os
    import time
    import torch.distributed as dist
    rank, local = int(os.environ["RANK"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("gloo")
    layer = None
    if os.environ.get("H2D_WITH_LAYER") == "1":  # the e2e process state: NCCL comm, IPC peer maps
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2206_03382_b200 import LayerState, MoELayerConfig
        W = int(os.environ["WORLD_SIZE"])
        cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=8 * W, model_dim=1024,
                             hidden_dim=4096, tokens_per_step=65536, top_k=1)
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        layer = LayerState.init(cfg, 402, rank=rank, device=local, nccl_id=obj[0])
    n = n_mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    o = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    e = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(dev), torch.cuda.Stream(dev)
    for dirs in (("h2d",), ("d2h",), ("h2d", "d2h")):
        for it in range(2):
            dist.barrier()
            t0 = time.perf_counter()
            for _ in range(reps):
                if "h2d" in dirs:
                    with torch.cuda.stream(s1):
                        d.copy_(h, non_blocking=True)
                if "d2h" in dirs:
                    with torch.cuda.stream(s2):
                        o.copy_(e, non_blocking=True)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
        print(f"rank {rank} {'+'.join(dirs):8s} {reps * n * len(dirs) / el / 1e9:7.1f} GB/s", flush=True)
    if layer is not None:
        layer.close()
    dist.destroy_process_group()


if __name__ == "__main__" and "RANK" in __import__("os").environ:
    run_ranks()
