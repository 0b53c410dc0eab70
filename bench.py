#!/usr/bin/env python3
"""Benchmark: MoE layer tokens/s (fwd+bwd) on B200, per BASELINE.json's metric.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload W]

N=1: the north-star SwinV2-MoE-B layer "TGT" (E=32, k=1, f=1.0, M=1024, V=4096, 32K tokens,
bf16). N>1 (torchrun, one rank per GPU, NCCL): expert parallelism with the configs[3] per-GPU
shape -- 8 experts and 64K tokens per GPU (E = 8N), flexible all-to-all + capacity pipelining --
so per-GPU work is fixed as N grows (weak scaling).

A step = gate -> encode -> dispatch -> expert FFN -> combine -> decode, then the full backward
(dx and every expert dW), on synthetic inputs drawn with the reference Rng(402) recipe on the
device. Timing: W untimed warm-up steps, barrier + synchronize, CUDA events around exactly K
steps, max over ranks. The per-step working set (weights 512 MiB + activations > 1 GiB per GPU)
is far larger than the 126 MB L2, so no explicit flush is needed between steps.

--impl reference times the reference algorithm on the host CPU: the fp64 oracle restatement
(oracle/, "port") because the C++ reference needs Eigen, absent from this image; rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    # name: (E, k, f, M, V, tokens per GPU, bpr, dtype)
    "TGT": dict(E=32, k=1, f=1.0, M=1024, V=4096, T=32768, bpr=False, dtype="bf16",
                desc="SwinV2-MoE-B layer (north-star target): E=32 k=1 f=1.0 M=1024 H=4096 32K tokens"),
    "C1": dict(E=8, k=1, f=1.0, M=512, V=2048, T=4096, bpr=False, dtype="f32",
               desc="configs[0]: single MoE layer fp32 E=8 k=1 f=1.0 M=512 H=2048 4096 tokens"),
    "C2": dict(E=32, k=1, f=1.0, M=768, V=3072, T=32768, bpr=False, dtype="bf16",
               desc="configs[1]: SwinV2-MoE-S layer E=32 k=1 f=1.0 M=768 H=3072 32K tokens"),
    "C3": dict(E=32, k=2, f=1.25, M=1024, V=4096, T=32768, bpr=True, dtype="bf16",
               desc="configs[2]: SwinV2-MoE-B top-2 + BPR E=32 k=2 f=1.25 M=1024 H=4096 32K tokens"),
    "C4": dict(E=8, k=1, f=1.0, M=1024, V=4096, T=65536, bpr=False, dtype="bf16",
               desc="configs[3] per GPU: 8 experts/GPU (E=8N) k=1 f=1.0 M=1024 H=4096 64K tokens/GPU"),
}
SEED = 402


def load_peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return dict(hbm=d["hbm_gbs"], bf16=d["bf16_tflops"], bf16_sus=d["bf16_tflops_sustained"],
                    source="measured (MEASURED_PEAKS.json)")
    return dict(hbm=6650.0, bf16=1590.0, bf16_sus=1400.0, source="fallback (B200_PROFILING.md)")


def fp64_gemm_peak(dev) -> float:
    """fp64 GEMM TF/s of this GPU (cuBLAS DGEMM, 8192^3, best of 5): the fp32 layer's roofline."""
    import torch
    n = 8192
    a = torch.rand(n, n, dtype=torch.float64, device=dev)
    b = torch.rand(n, n, dtype=torch.float64, device=dev)
    torch.matmul(a, b)
    best = None
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        ms = e0.elapsed_time(e1)
        best = ms if best is None else min(best, ms)
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


class ClockSampler:
    """SM clocks + throttle reasons sampled DURING the timed region: an NVML thread polling every
    2 ms (nvidia_ml_py), else `nvidia-smi -lms 50` (few samples in a sub-second region)."""
    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, device: int):
        self.device = self.smi_id(device)
        self.proc = None
        self.thread = None
        self.sm, self.mx, self.reasons, self.lines = [], 0.0, set(), []

    @staticmethod
    def smi_id(local: int) -> str:
        """nvidia-smi's id of CUDA device `local`: its UUID (robust to CUDA_VISIBLE_DEVICES
        remapping), else the CUDA_VISIBLE_DEVICES entry, else the index itself."""
        try:
            import torch
            u = str(torch.cuda.get_device_properties(local).uuid)
            if u:
                return u if u.startswith("GPU-") else "GPU-" + u
        except Exception:
            pass
        vis = os.environ.get("CUDA_VISIBLE_DEVICES", "")
        ids = [v.strip() for v in vis.split(",") if v.strip()]
        if local < len(ids):
            return ids[local]
        return str(local)

    def _nvml_start(self) -> bool:
        try:
            import threading
            import pynvml as N
            N.nvmlInit()
            h = (N.nvmlDeviceGetHandleByUUID(self.device) if self.device.startswith("GPU-")
                 else N.nvmlDeviceGetHandleByIndex(int(self.device)))
            self.mx = float(N.nvmlDeviceGetMaxClockInfo(h, N.NVML_CLOCK_SM))
            get_reasons = getattr(N, "nvmlDeviceGetCurrentClocksEventReasons",
                                  getattr(N, "nvmlDeviceGetCurrentClocksThrottleReasons", None))
            bits = [getattr(N, "nvmlClocksEventReason" + n, getattr(N, "nvmlClocksThrottleReason" + n, 0))
                    for n in ("HwSlowdown", "HwThermalSlowdown", "SwThermalSlowdown", "SwPowerCap")]
            self.stop = threading.Event()

            def loop():
                while not self.stop.is_set():
                    try:
                        self.sm.append(float(N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM)))
                        r = get_reasons(h) if get_reasons else 0
                        for name, b in zip(self.NAMES, bits):
                            if b and r & b:
                                self.reasons.add(name)
                    except Exception:
                        pass
                    self.stop.wait(0.002)

            self.thread = threading.Thread(target=loop, daemon=True)
            self.thread.start()
            return True
        except Exception:
            return False

    def __enter__(self):
        if self._nvml_start():
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "50", "-i", self.device],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except (FileNotFoundError, OSError):
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.thread is not None:
            self.stop.set()
            self.thread.join(timeout=2)
            return
        if self.proc is not None:
            time.sleep(0.06)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()
                out, _ = self.proc.communicate()
            self.lines = [ln for ln in out.splitlines() if ln.strip()]
            for ln in self.lines:
                parts = [p.strip() for p in ln.split(",")]
                if len(parts) < 6:
                    continue
                try:
                    self.sm.append(float(parts[0]))
                    self.mx = max(self.mx, float(parts[1]))
                except ValueError:
                    continue
                for n, v in zip(self.NAMES, parts[2:6]):
                    if v.lower().startswith("active"):
                        self.reasons.add(n)

    def summary(self) -> dict:
        return {"sm_mhz": statistics.median(self.sm) if self.sm else None,
                "sm_max_mhz": self.mx or None, "reasons": sorted(self.reasons),
                "samples": len(self.sm), "source": "nvml" if self.thread is not None else "nvidia-smi"}


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


def pick_workload(args, world):
    if args.workload:
        return args.workload
    return "TGT" if world == 1 else "C4"


def layer_dims(wl: str, world: int) -> dict:
    d = dict(WORKLOADS[wl])
    if wl == "C4":
        d["E"] = 8 * world
    elif world > 1:
        d["E"] = d["E"] * world  # same per-GPU expert count
    return d


# ------------------------------------------------------------------ CPU reference leg
def prepare_cpu(d: dict, sample_tokens: int):
    """Inputs for the fp64 oracle (the reference algorithm restated in C, OpenMP) on a token
    sample of the same layer; returns a callable running one fwd+bwd sample."""
    import numpy as np
    import oracle
    from paper_2206_03382_b200 import rng
    E, k, f, M, V = d["E"], d["k"], d["f"], d["M"], d["V"]
    T = sample_tokens
    off = rng.draw_offsets(M, E, V, 1, T)
    wg = rng.uniform(SEED, off["wg"], M * E).reshape(M, E)
    w1 = np.empty((E, M, V))
    w2 = np.empty((E, V, M))
    for e in range(E):
        o = off["experts"] + e * off["expert_stride"]
        w1[e] = rng.round_dtype(rng.uniform(SEED, o, M * V, -0.5, 0.5), d["dtype"]).reshape(M, V)
        w2[e] = rng.round_dtype(rng.uniform(SEED, o + M * V, V * M, -0.5, 0.5),
                                d["dtype"]).reshape(V, M)
    x = rng.round_dtype(rng.uniform(SEED, off["x"], T * M), d["dtype"]).reshape(T, M)
    dy = rng.round_dtype(rng.uniform(SEED, off["x"] + T * M, T * M), d["dtype"]).reshape(T, M)

    # every host core: torchrun sets OMP_NUM_THREADS=1 per rank, but only rank 0 runs this leg
    oracle.set_num_threads(len(os.sched_getaffinity(0)))

    def run():
        oracle.layer_step(x, wg, w1, w2, dy, 1, k, 0, f, d["bpr"])
    return run, oracle.num_threads()


def cpu_reference(d: dict, sample_tokens: int, min_seconds: float, max_iters: int):
    run, threads = prepare_cpu(d, sample_tokens)
    run()  # warm
    iters, t0 = 0, time.perf_counter()
    while True:
        run()
        iters += 1
        el = time.perf_counter() - t0
        if el >= min_seconds or iters >= max_iters:
            break
    return sample_tokens * iters / el, threads, el, iters


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return 0
    wl = pick_workload(args, world)
    d = layer_dims(wl, world)
    # bounded per-step sample so a --steps 50 run stays within a few minutes: 2 048 tokens
    # (~2.4 s/step at N=1 TGT on 16 host cores); at N=8 (C4, E=64) the per-step cost is dominated
    # by the E full-size fp64 dW the reference's backward writes (4.3 GB), so 1 024 tokens there
    sample = 2048 if world < 8 else 1024
    run, threads = prepare_cpu(d, sample)
    for _ in range(args.warmup):
        run()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        run()
    el = time.perf_counter() - t0
    value = sample * args.steps / el
    line = {
        "impl": "reference", "metric": "MoE layer tokens/s (fwd+bwd)", "value": value,
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": el / args.steps * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (reference Rng(402) draw order)",
        "config": {"workload": wl, "desc": d["desc"], "E": d["E"], "k": d["k"], "f": d["f"],
                   "M": d["M"], "V": d["V"], "tokens_per_gpu": d["T"], "bpr": d["bpr"],
                   "parallelism": f"ep{world}"},
        "cpu_baseline": {"value": value, "unit": "tokens/s", "cores": threads, "kind": "port",
                         "sample": f"{sample} of {d['T']} tokens per step (same E, k, f, M, V; "
                                   f"capacity scales with tokens), fp64 oracle restatement "
                                   f"(reference needs Eigen 3, absent)"},
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    emit(line)
    return 0


# ------------------------------------------------------------------ GPU leg
class StdoutToStderr:
    """Keeps library chatter (e.g. NCCL's version banner) off stdout: only the JSON line goes
    to the real stdout."""

    def __enter__(self):
        sys.stdout.flush()
        self.saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *a):
        sys.stdout.flush()
        os.dup2(self.saved, 1)
        os.close(self.saved)


def emit(line: dict) -> None:
    os.write(1, (json.dumps(line) + "\n").encode())


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default=None, choices=sorted(WORKLOADS))
    ap.add_argument("--degree", type=int, default=0, help="pipelining degree (0: adaptive Alg. 1)")
    ap.add_argument("--a2a", default="peer", choices=["peer", "nccl"],
                    help="W>1 all-to-all: copy engines over NVLink peer memory, or NCCL")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--update-weights", action="store_true",
                    help="training-loop variant: declare the expert weights changed every step "
                         "(moe_weights_updated, as after an on-device optimizer step), so every "
                         "forward rebuilds the ReLU certificate's W1^T copy and column norms")
    ap.add_argument("--no-phase-events", action="store_true",
                    help="A/B: time the steps without the per-phase CUDA events (no roofline)")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    args.warmup = max(args.warmup, 3)
    with StdoutToStderr():
        line = run_gpu(args)
    if line is not None:
        emit(line)
    return 0


def run_gpu(args):
    import torch
    import torch.distributed as dist

    from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward, ops, rng
    from paper_2206_03382_b200 import layer as L

    rank, local, world = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    wl = pick_workload(args, world)
    d = layer_dims(wl, world)
    E, k, f, M, V, T = d["E"], d["k"], d["f"], d["M"], d["V"], d["T"]
    tdt = torch.bfloat16 if d["dtype"] == "bf16" else torch.float32
    esz = 2 if d["dtype"] == "bf16" else 4

    nccl_id = None
    if world > 1:
        obj = [LayerState.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]
    adaptive = world > 1 and args.degree == 0
    cfg = MoELayerConfig(world_size=world, gpus_per_node=world, global_experts=E, model_dim=M,
                         hidden_dim=V, tokens_per_step=T, top_k=k, capacity_factor=f,
                         bpr=d["bpr"], dtype=d["dtype"], adaptive=adaptive,
                         degree=args.degree if args.degree else 1, a2a_backend=args.a2a)
    state = LayerState.init(cfg, SEED, rank=rank, device=local, nccl_id=nccl_id)
    off = rng.draw_offsets(M, E, V, world, T)
    x = torch.empty(T, M, dtype=tdt, device=dev)
    dy = torch.empty(T, M, dtype=tdt, device=dev)
    ops.fill_uniform(x, SEED, off["x"] + rank * T * M)
    ops.fill_uniform(dy, SEED, off["dy"] + rank * T * M)
    y = torch.empty_like(x)
    dx = torch.empty_like(x)
    dw1 = torch.empty(cfg.local_experts, M, V, dtype=torch.float32, device=dev)
    dw2 = torch.empty(cfg.local_experts, V, M, dtype=torch.float32, device=dev)

    def step():
        res = forward(state, x, y)
        backward(state, res.saved, dy, dx, dw1, dw2)
        if args.update_weights:
            state.weights_updated()

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # Alg. 1 explores its strategy space (2 forward steps per strategy: the first, cold one is not
    # recorded) before exploiting; let that finish
    # in the untimed warm-up so the timed steps run the chosen pipelining degree.
    for _ in range(args.warmup + (20 if adaptive else 0)):  # Alg. 1: 4 candidates x (1 + 3) forwards
        step()
    barrier()
    state.take_profile()  # drop warm-up records
    stream = torch.cuda.current_stream(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    # Pass 1 (the headline): K steps with no per-kernel events in the stream -- an event record
    # between two kernels keeps the next launch from overlapping the previous kernel's drain
    # (~45 us/step at TGT).
    with ClockSampler(local) as clk:
        barrier()
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        ev1.synchronize()
    ms = ev0.elapsed_time(ev1)
    # Pass 2 (the roofline / phase breakdown): the same K steps with CUDA events around every
    # kernel on the stream it runs on.
    prof = None
    if not args.no_phase_events:
        barrier()
        state.set_profiling(True)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        state.set_profiling(False)
        prof = state.take_profile()
    if prof is None:
        from paper_2206_03382_b200._lib import PHASES
        prof = {n: (0.0, 0) for n in PHASES}
    # Pass 3 (the GEMM roofline): the same K steps with no events; each tcgen05 GEMM records its
    # span on the device clock (%globaltimer, first CTA past the launch-dependency wait to the
    # last CTA's exit), so programmatic dependent launch overlaps the kernels as in pass 1.
    spans = None
    if not args.no_phase_events:
        barrier()
        state.set_kernel_spans(True)
        for _ in range(args.steps):
            step()
        torch.cuda.synchronize()
        spans = state.take_kernel_spans()
        state.set_kernel_spans(False)
    launches_per_step = state.kernel_launches()
    metrics = state.metrics()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * T / (ms_step * 1e-3)

    # roofline: expert GEMMs (tensor-bound) -- 12 * rows * M * V per step over capacity rows
    peaks = load_peaks()
    # event-timed ~0.2 ms kernels: the burst peak is the denominator (B200_PROFILING.md); the
    # sustained-peak fraction is reported beside it
    gemm_peak, gemm_bound = peaks["bf16"], "tensor"
    gemm_peak_sus = peaks["bf16_sus"]
    gemm_peak_src = peaks["source"] + " bf16_tflops (burst); frac_sustained uses bf16_tflops_sustained"
    gemm_kernel = "gemm_bf16_kernel (tcgen05 expert GEMMs, 6 launches/step)"
    if d["dtype"] == "f32":
        # fp32 layer: SIMT GEMMs with fp64 accumulation (fp32 products are exact in fp64) -- the
        # denominator is the fp64 GEMM rate of this GPU, measured here with cuBLAS DGEMM
        gemm_peak, gemm_bound = fp64_gemm_peak(dev), "fp64"
        gemm_peak_sus = gemm_peak
        gemm_peak_src = "measured in this run: cuBLAS DGEMM 8192^3, best of 5"
        gemm_kernel = "gemm_dmma_f32_kernel (DMMA fp64-accumulated fp32 expert GEMMs)"
    cap = metrics.capacity
    rows = cfg.local_experts * world * cap  # capacity rows per GPU: dE * (W * dC)
    gemm_flops = 12.0 * rows * M * V
    gemm_names = ["gemm_up", "gemm_down", "gemm_dgrad_mask", "gemm_dgrad", "gemm_wgrad1",
                  "gemm_wgrad2"]
    gemm_ms_ev = sum(prof[n][0] for n in gemm_names) / args.steps
    gemm_launches = sum(prof[n][1] for n in gemm_names) / args.steps
    gemm_ms_span = (sum(spans[n][0] for n in gemm_names) / args.steps
                    if spans and sum(spans[n][1] for n in gemm_names) > 0 else None)
    gemm_ms = gemm_ms_span if gemm_ms_span else gemm_ms_ev
    achieved_tf = gemm_flops / (gemm_ms * 1e-3) / 1e12 if gemm_ms > 0 else None
    achieved_ev = gemm_flops / (gemm_ms_ev * 1e-3) / 1e12 if gemm_ms_ev > 0 else None
    # algorithmic GEMM operand bytes per step: each of the 6 GEMMs reads its two operands and
    # writes its output once (rows x M / rows x V activations in the layer dtype, weights, fp32 dW)
    alg_bytes = float(rows * (M + V) * esz * 6 + cfg.local_experts * M * V * (esz * 4 + 4 * 2))
    traffic = None
    tp = ROOT / "profiles" / "ncu_traffic.json"
    if tp.exists():
        try:
            t = json.loads(tp.read_text()).get(wl)
            traffic = t["gemm_dram_bytes_per_step"] if t else None
        except Exception:
            traffic = None
    # dispatch/combine HBM rooflines (algorithmic bytes)
    drops = metrics.drop_count
    kept = T * k - drops
    slots = E * cap if world == 1 else E * cap  # encode writes every slot of every expert
    enc_bytes = (slots * M + kept * M) * esz + T * k * 8
    dec_bytes = (kept * M + T * M) * esz + T * k * 16
    enc_ms = prof["encode"][0] / args.steps
    dec_ms = prof["decode"][0] / args.steps
    dbwd_ms = prof["decode_bwd"][0] / args.steps
    ebwd_ms = prof["encode_bwd"][0] / args.steps
    gbs = lambda b, t: b / (t * 1e-3) / 1e9 if t > 0 else None  # noqa: E731
    fused_decode = bool(metrics.fused & 1)
    dispatch_stats = {"encode_gbs": gbs(enc_bytes, enc_ms), "decode_bwd_gbs": gbs(enc_bytes, dbwd_ms),
                      "hbm_peak_gbs": peaks["hbm"],
                      "encode_frac": (gbs(enc_bytes, enc_ms) or 0) / peaks["hbm"],
                      "decode_bwd_frac": (gbs(enc_bytes, dbwd_ms) or 0) / peaks["hbm"],
                      "fused": metrics.fused}
    if fused_decode:
        # decode / encode-backward run inside the down / dgrad GEMM epilogues (TMA row scatter);
        # the dropped tokens' zero rows are written by the encode / decode-backward passes
        dispatch_stats["decode"] = dispatch_stats["encode_bwd"] = "fused into GEMM epilogue"
    else:
        dispatch_stats.update({"decode_gbs": gbs(dec_bytes, dec_ms), "encode_bwd_gbs": gbs(dec_bytes, ebwd_ms),
                               "decode_frac": (gbs(dec_bytes, dec_ms) or 0) / peaks["hbm"]})
    phases_ms = {n: round(prof[n][0] / args.steps, 4) for n in prof}
    a2a_stats = None
    if world > 1:
        # dispatch (x rows forward, g*dy rows backward) = copy-engine pushes over NVLink: bytes this
        # rank sends off-GPU per step / the summed spans of its pushes (first block start -> last
        # block landed, CUDA events on the copy stream, phase pass)
        cc = -(-cap // max(1, metrics.degree))
        disp_bytes = 2.0 * (world - 1) * cfg.local_experts * metrics.degree * cc * M * esz
        xfer_ms = prof["xfer_dispatch"][0] / args.steps
        a2a_stats = {
            "transport": args.a2a, "dispatch_bytes_per_step": disp_bytes,
            "dispatch_xfer_ms_per_step": xfer_ms,
            "dispatch_gbs": gbs(disp_bytes, xfer_ms) if args.a2a == "peer" else None,
            "nvlink_peak_gbs": 900.0, "peak_source": "nominal NVLink 5 per direction per GPU",
            "combine": "fused into the down / dgrad GEMM epilogues (NVLink TMA stores)"
                       if metrics.fused & 2 else "copy-engine pushes",
            "note": "dispatch spans overlap the previous part's GEMM; a2a_fwd / a2a_bwd phases are "
                    "comm-stream spans incl. waits"}
        if a2a_stats["dispatch_gbs"]:
            a2a_stats["frac"] = a2a_stats["dispatch_gbs"] / 900.0

    # end to end through the host-buffer C ABI (H2D of x, dy and D2H of y, dx every step)
    e2e = None
    if not args.no_e2e:
        xh = x.cpu().pin_memory()
        dyh = dy.cpu().pin_memory()
        yh = torch.empty_like(xh).pin_memory()
        dxh = torch.empty_like(xh).pin_memory()
        # pipelined host API: step i+1's upload and step i's download overlap the compute
        for _ in range(2):
            L.forward_host_async(state, xh, yh)
            L.backward_host_async(state, dyh, dxh)
        L.host_sync(state)
        # three timed windows, the median reported (a single window is exposed to one-off host
        # hiccups: page-cache / scheduler noise on the box's shared host cores)
        n_e2e = max(3, args.steps // 2)
        windows = []
        for _ in range(3):
            barrier()
            t0 = time.perf_counter()
            for _ in range(n_e2e):
                L.forward_host_async(state, xh, yh)
                L.backward_host_async(state, dyh, dxh)
            L.host_sync(state)
            torch.cuda.synchronize()
            el = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([el], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                el = float(t.item())
            windows.append(el)
        el = sorted(windows)[1]
        e2e = {"value": world * T * n_e2e / el, "unit": "tokens/s",
               "windows_tokens_per_s": [round(world * T * n_e2e / w) for w in windows],
               "h2d_bytes_per_step": 2 * T * M * esz, "d2h_bytes_per_step": 2 * T * M * esz,
               "steps": n_e2e,
               "api": "moe_forward_host_async + moe_backward_host_async + moe_host_sync (C ABI, "
                      "pinned host buffers; uploads/downloads overlap neighbouring steps)"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        sample = max(256, T // 16)
        v, thr, el, it = cpu_reference(d, sample, 10.0, 50)
        cpu = {"value": v, "unit": "tokens/s", "cores": thr, "kind": "port",
               "sample": f"{it} x {sample}-token fwd+bwd samples of {wl} ({el:.1f} s), fp64 oracle "
                         f"restatement of the reference (Eigen absent, reference unbuildable)"}

    if rank == 0:
        line = {
            "metric": "MoE layer tokens/s (fwd+bwd)", "value": value, "unit": "tokens/s",
            "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": d["dtype"], "data": "synthetic (reference Rng(402) draw order, on device)",
            "config": {"workload": wl, "desc": d["desc"], "E": E, "k": k, "f": f, "M": M, "V": V,
                       "tokens_per_gpu": T, "global_batch": world * T, "bpr": d["bpr"],
                       "capacity": cap, "parallelism": f"ep{world}",
                       "a2a": args.a2a if world > 1 else None,
                       "degree": metrics.degree, "adaptive": adaptive,
                       "update_weights": bool(args.update_weights),
                       "l2": "per-step working set >1 GiB/GPU >> 126 MB L2 (no flush needed)"},
            "roofline": {"bound": gemm_bound, "achieved": achieved_tf, "peak": gemm_peak,
                         "unit": "TFLOP/s",
                         "frac": achieved_tf / gemm_peak if achieved_tf else None,
                         "frac_sustained": achieved_tf / gemm_peak_sus if achieved_tf else None,
                         "traffic": traffic / 6.0 if traffic else None,
                         "traffic_unit": "DRAM bytes per GEMM launch (mean of the 6 launches of a step)",
                         "traffic_per_step": traffic,
                         "traffic_source": "static: profiles/ncu_traffic.json (dram__bytes_read.sum + "
                                           "dram__bytes_write.sum from one ncu --set full capture of "
                                           "this workload; not re-measured in this run)" if traffic else None,
                         "algorithmic_bytes_per_step": alg_bytes,
                         "kernel": gemm_kernel,
                         "algorithmic": f"12*rows*M*V per step, rows={rows} capacity rows/GPU",
                         "gemm_ms_per_step": gemm_ms, "gemm_launches_per_step": gemm_launches,
                         "gemm_ms_per_step_event_timed": gemm_ms_ev,
                         "achieved_event_timed": achieved_ev,
                         "gemm_span_ms_per_step": ({n: spans[n][0] / args.steps for n in gemm_names}
                                                   if gemm_ms_span else None),
                         "gemm_effective_sm_mhz": (spans["_sm_mhz"][0] if gemm_ms_span else None),
                         "peak_source": gemm_peak_src,
                         "timing": ("device-clock kernel spans (%globaltimer, first CTA past the "
                                    "launch-dependency wait to the last CTA exit) over a third "
                                    "event-free K-step pass; achieved_event_timed: CUDA events "
                                    "around every GEMM launch (second pass; events stop "
                                    "programmatic dependent launch, so each launch pays its "
                                    "prologue and drain)") if gemm_ms_span else
                                   "CUDA events around every GEMM launch over a second K-step "
                                   "pass (the headline value comes from an event-free pass)"},
            "dispatch": dispatch_stats,
            "a2a": a2a_stats,
            "phases_ms": phases_ms,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clk.summary(),
            "drop_count": drops,
            "relu_fixups_last_chunk": metrics.relu_fixups,
        }
    else:
        line = None
    if world > 1:
        dist.barrier()
        dist.destroy_process_group()
    state.close()
    return line


if __name__ == "__main__":
    sys.exit(main())
