"""Capacity-factor x pipelining-degree sweep (BASELINE.json configs[4]) on W GPUs, with the
adaptive switch (Alg. 1) beside the fixed degrees.

    torchrun --nproc-per-node W --master-addr 127.0.0.1 tools/sweep.py [--out FILE]

Per GPU the configs[3] shape (8 experts/GPU, E = 8W, k=1, M=1024, H=4096, 64K tokens/GPU,
bf16). For every f in {0.5, 0.625, 1.0, 1.25} and degree in {1, 2, 4, 8}: fwd+bwd step time
(CUDA events around K steps, max over ranks) and the forward time alone. Then one adaptive layer
walks the same f values through moe_set_capacity_factor: Alg. 1 explores each f's strategies in
the warm-up and the timed steps run the degree it settled on."""
import argparse
import json
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward, ops, rng  # noqa: E402

FS = (0.5, 0.625, 1.0, 1.25)
DEGREES = (1, 2, 4, 8)
SEED = 402


def timed(fn, steps, dev, world):
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    dist.barrier()
    torch.cuda.synchronize()
    ev0.record()
    for _ in range(steps):
        fn()
    ev1.record()
    ev1.synchronize()
    t = torch.tensor([ev0.elapsed_time(ev1) / steps], device=dev, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=4)
    ap.add_argument("--tokens", type=int, default=65536)
    ap.add_argument("--out", default=None)
    ap.add_argument("--fs", default=",".join(map(str, FS)))
    ap.add_argument("--degrees", default=",".join(map(str, DEGREES)))
    ap.add_argument("--phases", action="store_true", help="also print per-kernel times")
    args = ap.parse_args()
    fs = tuple(float(v) for v in args.fs.split(","))
    degrees = tuple(int(v) for v in args.degrees.split(","))
    rank, W, local = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"]), int(os.environ["LOCAL_RANK"])
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", device_id=dev)
    E, M, V, T = 8 * W, 1024, 4096, args.tokens
    off = rng.draw_offsets(M, E, V, W, T)
    x = torch.empty(T, M, dtype=torch.bfloat16, device=dev)
    dy = torch.empty_like(x)
    ops.fill_uniform(x, SEED, off["x"] + rank * T * M)
    ops.fill_uniform(dy, SEED, off["dy"] + rank * T * M)
    y, dx = torch.empty_like(x), torch.empty_like(x)
    dw1 = torch.empty(8, M, V, dtype=torch.float32, device=dev)
    dw2 = torch.empty(8, V, M, dtype=torch.float32, device=dev)

    def make(f, degree, adaptive):
        cfg = MoELayerConfig(world_size=W, gpus_per_node=W, global_experts=E, model_dim=M,
                             hidden_dim=V, tokens_per_step=T, top_k=1, capacity_factor=f,
                             dtype="bf16", adaptive=adaptive, degree=degree)
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        return LayerState.init(cfg, SEED, rank=rank, device=local, nccl_id=obj[0])

    def measure(st, warm):
        saved = {}

        def step():
            res = forward(st, x, y)
            backward(st, res.saved, dy, dx, dw1, dw2)

        def fwd():
            saved["r"] = forward(st, x, y)

        for _ in range(warm):
            step()
        ms = timed(step, args.steps, dev, W)
        ms_f = timed(fwd, args.steps, dev, W)
        m = st.metrics()
        extra = {}
        if args.phases:
            torch.cuda.synchronize()
            st.take_profile()
            st.set_profiling(True)
            for _ in range(args.steps):
                step()
            torch.cuda.synchronize()
            st.set_profiling(False)
            extra["phases_ms"] = {n: round(v[0] / args.steps, 4) for n, v in st.take_profile().items()}
        return dict(**extra, ms_step=ms, ms_fwd=ms_f, tokens_per_s=W * T / (ms * 1e-3),
                    capacity=m.capacity, degree=m.degree)

    rows = []
    for f in fs:
        for deg in degrees:
            st = make(f, deg, False)
            r = measure(st, args.warmup)
            st.close()
            r.update(f=f, mode=f"fixed d={deg}")
            rows.append(r)
            if rank == 0:
                print(json.dumps(r), file=sys.stderr, flush=True)
    st = make(fs[0], 1, True)
    for f in fs:
        st.set_capacity_factor(f)
        # Alg. 1: 4 strategies x 2 forward executions (the first one cold) before it exploits
        r = measure(st, args.warmup + 12)
        r.update(f=f, mode="adaptive")
        rows.append(r)
        if rank == 0:
            print(json.dumps(r), file=sys.stderr, flush=True)
    st.close()
    if rank == 0:
        out = {"world": W, "shape": f"E={E} (8/GPU) k=1 M={M} H={V} {T} tokens/GPU bf16",
               "steps": args.steps, "timing": "CUDA events over K steps, max over ranks",
               "rows": rows}
        best = {}
        for r in rows:
            if r["mode"].startswith("fixed"):
                b = best.get(r["f"])
                if b is None or r["ms_step"] < b["ms_step"]:
                    best[r["f"]] = r
        out["summary"] = [
            {"f": f, "best_fixed": best[f]["mode"], "best_ms": best[f]["ms_step"],
             "adaptive_degree": a["degree"], "adaptive_ms": a["ms_step"],
             "adaptive_vs_best": best[f]["ms_step"] / a["ms_step"]}
            for f in fs for a in rows if a["mode"] == "adaptive" and a["f"] == f]
        s = json.dumps(out, indent=1)
        print(s)
        if args.out:
            with open(args.out, "w") as fh:
                fh.write(s + "\n")
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
