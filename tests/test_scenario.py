"""Scenario runner / records.csv compatibility: the reference's own bench tests
(/root/reference/proj/tests/test_bench.cpp) restated against paper_2206_03382_b200.scenario."""
import math

import pytest
import torch

from paper_2206_03382_b200 import scenario as S


def test_workload_traces_deterministic_and_in_range():
    """test_bench.cpp:9-38."""
    assert S.generate_workload_trace(S.TraceSpec("constant", f=2.0), 5, 1) == [2.0] * 5
    cy = S.generate_workload_trace(S.TraceSpec("cycle", values=[1.0, 2.0, 4.0]), 7, 1)
    assert cy == [1.0, 2.0, 4.0, 1.0, 2.0, 4.0, 1.0]
    rnd = S.TraceSpec("random", f_min=0.5, f_max=4.0)
    r1 = S.generate_workload_trace(rnd, 50, 9)
    assert r1 == S.generate_workload_trace(rnd, 50, 9)
    assert r1 != S.generate_workload_trace(rnd, 50, 10)
    assert all(0.5 <= f <= 4.0 for f in r1)
    with pytest.raises(ValueError):
        S.generate_workload_trace(S.TraceSpec("cycle"), 3, 1)
    with pytest.raises(ValueError):
        S.generate_workload_trace(S.TraceSpec("constant", f=2.0), 0, 1)


def test_random_trace_is_the_reference_rng_stream():
    """Rng(seed).uniform(f_min, f_max), core.cpp:66-83: draw n (1-based) = mix(seed + n phi)."""
    seed = 9
    st = seed
    want = []
    for _ in range(3):
        st = (st + S.PHI) & S.MASK64
        z = st
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & S.MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & S.MASK64
        z ^= z >> 31
        want.append(0.5 + 3.5 * ((z >> 11) * 2.0 ** -53))
    got = S.generate_workload_trace(S.TraceSpec("random", f_min=0.5, f_max=4.0), 3, seed)
    assert got == want


def test_scenario_grid_expands_row_major():
    """test_bench.cpp:40-63."""
    sc = S.parse_scenario_text('''{
      "name": "sweep", "steps": 3, "seed": 7,
      "grid": {"world_size": [2, 4], "gpus_per_node": [2], "tokens_per_step": [8],
               "model_dim": [4], "hidden_dim": [8], "top_k": [1], "experts_per_rank": [1, 2]},
      "trace": {"kind": "cycle", "values": [1.0, 2.0]},
      "strategy": "adaptive", "parallel": "p1"}''')
    assert (sc.name, sc.steps, sc.seed) == ("sweep", 3, 7)
    assert len(sc.settings) == 4
    assert sc.settings[0].id == "sweep#0"
    assert sc.settings[0].dims.world_size == 2 and sc.settings[0].dims.global_experts == 2
    assert sc.settings[1].dims.global_experts == 4  # experts_per_rank varies fastest
    assert sc.settings[2].dims.world_size == 4
    assert sc.adaptive and sc.parallel == "p1" and sc.trace.kind == "cycle"


def test_scenario_fractional_placement():
    """test_bench.cpp:65-73."""
    sc = S.parse_scenario_text('{"grid": {"world_size": [4], "experts_per_rank": [0.5], "top_k": [1]}}')
    d = sc.settings[0].dims
    assert d.is_sharded and d.ranks_per_expert == 2 and d.global_experts == 2


def test_scenario_parse_errors():
    """test_bench.cpp:75-85: malformed input raises invalid_argument with a line diagnostic."""
    with pytest.raises(ValueError, match="line 2"):
        S.parse_scenario_text('{\n  "steps": oops\n}')
    with pytest.raises(ValueError, match="steps"):
        S.parse_scenario_text('{"steps": 0}')
    with pytest.raises(ValueError, match="non-empty"):
        S.parse_scenario_text('{"grid": {"world_size": []}}')
    with pytest.raises(ValueError):
        S.parse_scenario_text('{"grid": {"experts_per_rank": [0.3]}}')
    with pytest.raises(ValueError):
        S.parse_scenario_text('{"parallel": "both"}')


def test_records_csv_round_trip():
    """test_bench.cpp:87-102."""
    recs = [S.StepRecord("a#0", 0, 1.0, 4, "linearx1", "p1", 1.25e-3, 4096.0, 2),
            S.StepRecord("a#0", 1, 2.5, 8, "2dhx4", "p2", 7.5e-4, 8192.0, 0)]
    csv = S.records_csv(recs)
    assert csv.split("\n")[0] == S.HEADER
    assert csv.split("\n")[1] == "a#0,0,1,4,linearx1,p1,0.00125,4096,2"
    back = S.parse_records_csv(csv)
    assert back[0].scenario_id == "a#0" and back[0].sim_seconds == 1.25e-3
    assert back[1].strategy == "2dhx4" and back[1].drop_count == 0
    with pytest.raises(ValueError):
        S.parse_records_csv("bogus\n")


def test_report():
    """emit_report (bench.cpp:301-353): best / worst strategy means, regret vs the per-f best."""
    recs = [S.StepRecord("s#0", 0, 1.0, 4, "linearx1", "p1", 2.0, 0.0, 0),
            S.StepRecord("s#0", 1, 1.0, 4, "linearx2", "p1", 1.0, 0.0, 0),
            S.StepRecord("s#0", 2, 2.0, 8, "linearx2", "p1", 3.0, 0.0, 0)]
    rep = S.emit_report(recs).split("\n")
    assert rep[0].startswith("scenario_id,steps,mean_s,best_strategy")
    # mean 2; per strategy: linearx1 2.0, linearx2 2.0 -> best is the first (map order), worst 2;
    # regret = (2 - 1) + 0 + 0 over 3; speedup vs baseline linearx1 = 2 / 2
    assert rep[1] == "s#0,3,2,linearx1,2,2,0.333333333333,1,1"


@pytest.mark.gpu
def test_materialized_run_on_gpu(cuda):
    """test_bench.cpp:104-121 on the GPU (W = 1 here; the W = 2 grid runs under torchrun):
    identical decisions across runs, capacity follows the f trace, measured seconds > 0."""
    sc = S.parse_scenario_text('''{
      "name": "tiny", "steps": 4, "seed": 11,
      "grid": {"world_size": [1, 2], "gpus_per_node": [1], "tokens_per_step": [64],
               "model_dim": [16], "hidden_dim": [32], "top_k": [1], "experts_per_rank": [4]},
      "trace": {"kind": "cycle", "values": [1.0, 2.0]}}''')
    a = S.run_scenario(sc, 64, "f32")
    b = S.run_scenario(sc, 64, "f32")
    assert len(a) == 4  # the W = 2 setting is skipped in a single process
    strip = lambda rs: [(r.scenario_id, r.step, r.f, r.capacity, r.strategy, r.drop_count) for r in rs]  # noqa: E731
    assert strip(a) == strip(b)
    assert a[0].f == 1.0 and a[1].f == 2.0 and a[0].capacity < a[1].capacity
    assert all(r.sim_seconds > 0.0 for r in a)
    back = S.parse_records_csv(S.records_csv(a))
    assert strip(back) == strip(a)
