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


if __name__ == "__main__":
    run()
