"""Scenario runner and `records.csv` compatibility (the reference's moe_bench).

Restates /root/reference/proj/src/bench.cpp and tools/moe_bench.cpp:
  parse_scenario_text      bench.cpp:98-185   (same JSON grammar, defaults, grid order, errors)
  generate_workload_trace  bench.cpp:65-96    (constant / cycle / random from Rng(seed))
  run_scenario             bench.cpp:189-268  (materialized path: per-step FixedCapacity{f}, x drawn
                                               after LayerState::init, forward, StepMetrics)
  records_csv / parse_records_csv / emit_report  bench.cpp:270-353 (byte-identical formats)

Differences, by design:
  * `sim_seconds` holds the *measured* forward time on the B200s (CUDA events, max over ranks).
  * The payload-free path (bench.cpp:222-248) evaluates the reference's fabric cost model, which is
    out of scope here; settings that cannot run on the launched GPUs (W larger than the process
    count or than `ranks_materialize_max`) are skipped with a note on stderr. Sharded placement
    (experts_per_rank < 1) and the parallel control (adaptive | p1 | p2) run on the GPUs.
  * The layer runs in `dtype` (bf16 or f32); x is drawn in fp64 by the reference Rng and rounded.

Usage (one process per GPU; W-rank settings use ranks 0..W-1):
  python -m paper_2206_03382_b200.scenario run scenario.json --out DIR [--seed S]
  torchrun --nproc-per-node N -m paper_2206_03382_b200.scenario run scenario.json --out DIR
  python -m paper_2206_03382_b200.scenario report DIR/records.csv
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
from dataclasses import dataclass, field
from pathlib import Path

from . import rng as _rng

PHI = 0x9E3779B97F4A7C15
MASK64 = (1 << 64) - 1
HEADER = "scenario_id,step,f,capacity,strategy,parallel,sim_seconds,comm_bytes,drop_count"


# ---------------------------------------------------------------- scenario model (bench.hpp)
@dataclass
class Dims:
    world_size: int
    gpus_per_node: int
    tokens_per_step: int
    model_dim: int
    hidden_dim: int
    top_k: int
    global_experts: int
    experts_per_rank: int = 0   # ExpertsPerRank{x} (0 when sharded)
    ranks_per_expert: int = 0   # RanksPerExpert{s} (0 when not sharded)

    @property
    def is_sharded(self) -> bool:
        return self.ranks_per_expert > 0


@dataclass
class ScenarioSetting:
    id: str
    dims: Dims


@dataclass
class TraceSpec:
    kind: str = "constant"  # constant | cycle | random
    f: float = 1.0
    values: list = field(default_factory=list)
    f_min: float = 1.0
    f_max: float = 1.0


@dataclass
class Scenario:
    name: str = "scenario"
    steps: int = 1
    seed: int = 1
    settings: list = field(default_factory=list)
    trace: TraceSpec = field(default_factory=TraceSpec)
    adaptive: bool = False           # StrategyControl defaults (moe_layer.hpp:12-15): linear x1
    degree: int = 1
    algo: str = "linear"
    parallel: str = "p1"             # adaptive | p1 | p2


@dataclass
class StepRecord:
    scenario_id: str
    step: int
    f: float
    capacity: int
    strategy: str
    parallel: str
    sim_seconds: float
    comm_bytes: float
    drop_count: int


def _fail(text: str, lineno: int, what: str):
    raise ValueError(f"scenario line {lineno}: {what}")


def _dims_validate(d: Dims) -> None:
    """Dims::validate (core.cpp:8-26)."""
    if d.world_size < 1 or d.gpus_per_node < 1:
        raise ValueError("Dims: W and m must be >= 1")
    if d.world_size % d.gpus_per_node:
        raise ValueError("Dims: world size must be a multiple of gpus per node")
    if d.top_k < 1 or d.top_k > d.global_experts:
        raise ValueError("Dims: need 1 <= k <= E")
    if d.model_dim < 1 or d.hidden_dim < 1 or d.tokens_per_step < 1:
        raise ValueError("Dims: M, V, T must be >= 1")
    if not d.is_sharded and d.hidden_dim % d.world_size:
        raise ValueError("ExpertParams: hidden dim must divide into parameter slices")


def make_dims(W, m, T, M, V, k, e) -> Dims:
    """bench.cpp:36-61 (experts_per_rank >= 1: integer x; < 1: 1/s with s | W)."""
    d = Dims(int(W), int(m), int(T), int(M), int(V), int(k), 0)
    if e >= 1.0:
        x = int(round(e))
        if float(x) != e:
            raise ValueError("experts_per_rank >= 1 must be an integer")
        d.experts_per_rank = x
        d.global_experts = d.world_size * x
    else:
        s = int(round(1.0 / e))
        if abs(1.0 / s - e) > 1e-12:
            raise ValueError("experts_per_rank < 1 must be 1/s for integer s")
        if d.world_size % s:
            raise ValueError("experts_per_rank 1/s needs s to divide world_size")
        d.ranks_per_expert = s
        d.global_experts = d.world_size // s
    _dims_validate(d)
    return d


def parse_scenario_text(text: str) -> Scenario:
    """bench.cpp:98-185: raises ValueError (the reference's invalid_argument) with a line
    diagnostic for malformed JSON."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        _fail(text, e.lineno, e.msg)
    if not isinstance(j, dict):
        raise ValueError("scenario: top level must be an object")
    sc = Scenario()
    sc.name = j.get("name", "scenario")
    sc.steps = j.get("steps", 1)
    sc.seed = j.get("seed", 1)
    if not isinstance(sc.steps, int) or sc.steps < 1:
        raise ValueError("steps must be >= 1")
    grid = j.get("grid", {})

    def gv(key, fallback):
        return [float(v) for v in grid[key]] if key in grid else fallback

    Ws, ms, Ts = gv("world_size", [4]), gv("gpus_per_node", [2]), gv("tokens_per_step", [16])
    Ms, Vs, ks, Es = gv("model_dim", [8]), gv("hidden_dim", [8]), gv("top_k", [2]), gv("experts_per_rank", [1])
    if not all((Ws, ms, Ts, Ms, Vs, ks, Es)):
        raise ValueError("grid lists must be non-empty")
    idx = 0
    for W in Ws:
        for m in ms:
            for T in Ts:
                for M in Ms:
                    for V in Vs:
                        for k in ks:
                            for e in Es:  # experts_per_rank varies fastest
                                sc.settings.append(ScenarioSetting(f"{sc.name}#{idx}",
                                                                   make_dims(W, m, T, M, V, k, e)))
                                idx += 1
    if "trace" in j:
        t = j["trace"]
        kind = t.get("kind", "constant")
        if kind == "constant":
            sc.trace = TraceSpec("constant", f=t.get("f", 1.0))
        elif kind == "cycle":
            sc.trace = TraceSpec("cycle", values=[float(v) for v in t.get("values", [])])
        elif kind == "random":
            sc.trace = TraceSpec("random", f_min=t.get("f_min", 1.0), f_max=t.get("f_max", 1.0))
        else:
            raise ValueError("trace kind must be constant|cycle|random")
    if "strategy" in j:
        s = j["strategy"]
        if s == "adaptive":
            sc.adaptive = True
        elif isinstance(s, dict):
            sc.adaptive = False
            sc.algo = s.get("algo", "linear")
            if sc.algo not in ("linear", "2dh"):
                raise ValueError("strategy algo must be linear|2dh")
            sc.degree = int(s.get("degree", 1))
        else:
            raise ValueError('strategy must be "adaptive" or an object')
    if "parallel" in j:
        p = j["parallel"]
        if p not in ("adaptive", "p1", "p2"):
            raise ValueError("parallel must be adaptive|p1|p2")
        sc.parallel = p
    return sc


def load_scenario(path) -> Scenario:
    try:
        text = Path(path).read_text()
    except OSError:
        raise ValueError(f"cannot open scenario file: {path}")
    return parse_scenario_text(text)


def generate_workload_trace(spec: TraceSpec, steps: int, seed: int) -> list:
    """bench.cpp:65-96: the random trace is Rng(seed).uniform(f_min, f_max) per step."""
    if steps < 1:
        raise ValueError("generate_workload_trace: steps must be >= 1")
    if spec.kind == "constant":
        if not spec.f > 0.0:
            raise ValueError("trace: constant f must be positive")
        return [float(spec.f)] * steps
    if spec.kind == "cycle":
        if not spec.values:
            raise ValueError("trace: cycle needs values")
        if any(not v > 0.0 for v in spec.values):
            raise ValueError("trace: cycle values must be positive")
        return [float(spec.values[i % len(spec.values)]) for i in range(steps)]
    if spec.kind == "random":
        if not spec.f_min > 0.0 or spec.f_max < spec.f_min:
            raise ValueError("trace: need 0 < f_min <= f_max")
        return [float(v) for v in _rng.uniform(seed, 0, steps, spec.f_min, spec.f_max)]
    raise ValueError("trace kind must be constant|cycle|random")


# ---------------------------------------------------------------- records.csv (bench.cpp:270-353)
def _fmt(v: float) -> str:
    """std::ostream << setprecision(12) << v (defaultfloat) == %.12g."""
    return f"{v:.12g}"


def records_csv(records) -> str:
    out = [HEADER]
    for r in records:
        out.append(f"{r.scenario_id},{r.step},{_fmt(r.f)},{r.capacity},{r.strategy},{r.parallel},"
                   f"{_fmt(r.sim_seconds)},{_fmt(r.comm_bytes)},{r.drop_count}")
    return "\n".join(out) + "\n"


def parse_records_csv(text: str) -> list:
    lines = text.split("\n")
    if not lines or lines[0] != HEADER:
        raise ValueError("records: missing or unexpected header")
    recs = []
    for line in lines[1:]:
        if not line:
            continue
        c = line.split(",")
        if len(c) != 9:
            raise ValueError(f"records: bad column count: {line}")
        recs.append(StepRecord(c[0], int(c[1]), float(c[2]), int(c[3]), c[4], c[5], float(c[6]),
                               float(c[7]), int(c[8])))
    return recs


def emit_report(records) -> str:
    """Per scenario id: steps, mean, best / worst strategy means, regret vs the per-f best,
    speedups (bench.cpp:301-353)."""
    if not records:
        raise ValueError("emit_report: no records")
    order, groups = [], {}
    for r in records:
        if r.scenario_id not in groups:
            groups[r.scenario_id] = []
            order.append(r.scenario_id)
        groups[r.scenario_id].append(r)
    out = ["scenario_id,steps,mean_s,best_strategy,best_mean_s,worst_mean_s,mean_regret_s,"
           "speedup_vs_worst,speedup_vs_baseline"]
    for sid in order:
        rs = groups[sid]
        per = {}
        best_by_f = {}
        total = 0.0
        for r in rs:
            acc = per.setdefault(r.strategy, [0.0, 0])
            acc[0] += r.sim_seconds
            acc[1] += 1
            if r.f not in best_by_f or r.sim_seconds < best_by_f[r.f]:
                best_by_f[r.f] = r.sim_seconds
            total += r.sim_seconds
        best_name, best_mean, worst_mean = "", 0.0, 0.0
        for i, name in enumerate(sorted(per)):  # std::map iteration order
            mean = per[name][0] / per[name][1]
            if i == 0 or mean < best_mean:
                best_mean, best_name = mean, name
            if i == 0 or mean > worst_mean:
                worst_mean = mean
        regret = sum(r.sim_seconds - best_by_f[r.f] for r in rs)
        n = float(len(rs))
        mean = total / n
        line = (f"{sid},{len(rs)},{_fmt(mean)},{best_name},{_fmt(best_mean)},{_fmt(worst_mean)},"
                f"{_fmt(regret / n)},{_fmt(worst_mean / mean)},")
        if "linearx1" in per:
            line += _fmt(per["linearx1"][0] / per["linearx1"][1] / mean)
        out.append(line)
    return "\n".join(out) + "\n"


# ---------------------------------------------------------------- materialized runs on the GPUs
def _setting_seed(base: int, i: int) -> int:
    return (base + PHI * (i + 1)) & MASK64


def runnable(d: Dims, parallel: str, world: int, ranks_materialize_max: int):
    """None if the setting runs here, else the reason it is skipped."""
    if d.world_size > ranks_materialize_max:
        return "payload-free path (fabric cost model) is out of scope"
    if d.world_size > world:
        return f"needs {d.world_size} GPU processes, {world} launched"
    return None


def run_scenario(sc: Scenario, ranks_materialize_max: int = 64, dtype: str = "f32",
                 rank: int = 0, world: int = 1, device: int = 0, log=sys.stderr) -> list:
    """bench.cpp:189-219 + 253-268 on the GPUs. Every process calls it (SPMD); records are
    returned on every rank. Settings with W < world run on ranks 0..W-1."""
    import torch
    from .layer import LayerState, MoELayerConfig, forward

    dist = None
    if world > 1:
        import torch.distributed as dist  # noqa: F811
    records = []
    for i, setting in enumerate(sc.settings):
        d = setting.dims
        why = runnable(d, sc.parallel, world, ranks_materialize_max)
        if why:
            if rank == 0:
                print(f"scenario: skip {setting.id} (W={d.world_size}): {why}", file=log)
            continue
        seed = _setting_seed(sc.seed, i)
        trace = generate_workload_trace(sc.trace, sc.steps, seed)
        W, T, M = d.world_size, d.tokens_per_step, d.model_dim
        active = rank < W
        cfg = MoELayerConfig(world_size=W, gpus_per_node=d.gpus_per_node,
                             global_experts=d.global_experts, model_dim=M,
                             hidden_dim=d.hidden_dim, tokens_per_step=T, top_k=d.top_k,
                             capacity="fixed", capacity_factor=trace[0], dtype=dtype,
                             adaptive=sc.adaptive, degree=sc.degree if not sc.adaptive else 1,
                             parallel=sc.parallel, a2a_algo=sc.algo if not sc.adaptive else "linear")
        nid = None
        if W > 1:
            obj = [LayerState.unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            nid = obj[0]
        recs = []
        if active:
            st = LayerState.init(cfg, seed, rank=rank, device=device, nccl_id=nid)
            off = _rng.draw_offsets(M, d.global_experts, d.hidden_dim, W, T)["x"]
            tdt = cfg.torch_dtype
            for step in range(sc.steps):
                st.set_capacity_factor(trace[step])
                # Tensor::random({W*T, M}, rng) after the init draws; this rank's block of rows
                base = off + step * W * T * M + rank * T * M
                x = torch.as_tensor(_rng.round_dtype(
                    _rng.uniform(seed, base, T * M).reshape(T, M), dtype)).to(tdt).to(f"cuda:{device}")
                forward(st, x)
                m = st.metrics()
                recs.append([step, m.f, m.capacity, m.degree, m.a2a_algo, m.seconds, m.comm_bytes,
                             m.drop_count, m.parallel])
            torch.cuda.synchronize()
            st.close()
        if W > 1:
            # whole-layer numbers: time = max over ranks, bytes and drops summed over ranks
            t = torch.zeros(sc.steps, 3, dtype=torch.float64, device=f"cuda:{device}")
            if active:
                for s_, r in enumerate(recs):
                    t[s_] = torch.tensor([r[5], r[6], r[7]], dtype=torch.float64)
            tmax = t[:, 0].clone()
            dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
            tsum = t[:, 1:].clone()
            dist.all_reduce(tsum)
            if not active:
                recs = [[s_, 0.0, 0, 0, "linear", 0.0, 0.0, 0, "p1"] for s_ in range(sc.steps)]
                meta = [None]
            else:
                meta = [[(r[1], r[2], r[3], r[4], r[8]) for r in recs]] if rank == 0 else [None]
            dist.broadcast_object_list(meta, src=0)
            for s_ in range(sc.steps):
                f, cap, deg, algo, par = meta[0][s_]
                recs[s_] = [s_, f, cap, deg, algo, float(tmax[s_]), float(tsum[s_, 0]),
                            int(round(float(tsum[s_, 1]))), par]
        for step, f, cap, deg, algo, secs, cbytes, drops, par in recs:
            records.append(StepRecord(setting.id, step, f, cap, f"{algo}x{deg}", par, secs,
                                      cbytes, drops))
    return records


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="moe_bench", description="MoE layer scenario runner (B200)")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="run a scenario file and write records.csv")
    r.add_argument("scenario")
    r.add_argument("--out", default=".")
    r.add_argument("--seed", type=int, default=-1, help="override the scenario seed")
    r.add_argument("--ranks-materialize-max", type=int, default=64)
    r.add_argument("--dtype", default="f32", choices=["f32", "bf16"])
    rep = sub.add_parser("report", help="summarize a records.csv")
    rep.add_argument("records")
    a = ap.parse_args(argv)
    try:
        if a.cmd == "report":
            sys.stdout.write(emit_report(parse_records_csv(Path(a.records).read_text())))
            return 0
        sc = load_scenario(a.scenario)
        if a.seed >= 0:
            sc.seed = a.seed
        world = int(os.environ.get("WORLD_SIZE", "1"))
        rank = int(os.environ.get("RANK", "0"))
        local = int(os.environ.get("LOCAL_RANK", "0"))
        if world > 1:
            import torch
            import torch.distributed as dist
            torch.cuda.set_device(local)
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        recs = run_scenario(sc, a.ranks_materialize_max, a.dtype, rank, world, local)
        if rank == 0:
            out = Path(a.out)
            out.mkdir(parents=True, exist_ok=True)
            (out / "records.csv").write_bytes(records_csv(recs).encode())
            print(f"wrote {len(recs)} records to {out / 'records.csv'}")
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return 0
    except (ValueError, RuntimeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
