"""Peer-copy bandwidth over NVLink (copy engines): one GPU pushing to 1..N-1 peers concurrently."""
import torch
n = torch.cuda.device_count()
for d in range(n):
    for e in range(n):
        if d != e:
            torch.cuda.set_device(d)
            assert torch.cuda.can_device_access_peer(d, e)
sizes = [8 << 20, 32 << 20, 128 << 20]
src = torch.empty(128 << 20, dtype=torch.uint8, device="cuda:0")
dst = {e: torch.empty(128 << 20, dtype=torch.uint8, device=f"cuda:{e}") for e in range(n)}
torch.cuda.set_device(0)
streams = {e: torch.cuda.Stream(device=0) for e in range(n)}
for npeers in range(1, n):
    for sz in sizes:
        for rep in range(2):
            ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(0)
            ev0.record()
            evs = []
            for e in range(1, npeers + 1):
                s = streams[e]
                s.wait_event(ev0)
                with torch.cuda.stream(s):
                    dst[e][:sz].copy_(src[:sz], non_blocking=True)
                x = torch.cuda.Event(); x.record(s); evs.append(x)
            for x in evs: torch.cuda.current_stream().wait_event(x)
            ev1.record(); torch.cuda.synchronize(0)
            ms = ev0.elapsed_time(ev1)
        print(f"peers={npeers} size={sz>>20}MB each: {ms*1e3:.0f} us, per-peer {sz/ms/1e6:.0f} GB/s, total {npeers*sz/ms/1e6:.0f} GB/s", flush=True)
# local D2D copy engine
d2 = torch.empty_like(src)
for sz in sizes:
    ev0 = torch.cuda.Event(enable_timing=True); ev1 = torch.cuda.Event(enable_timing=True)
    ev0.record(); d2[:sz].copy_(src[:sz]); ev1.record(); torch.cuda.synchronize()
    print(f"local copy_ {sz>>20}MB: {ev0.elapsed_time(ev1)*1e3:.0f} us")
