"""Writes tests/golden/reference_kats.json: the reference's own known-answer tests for the MoE
layer path, transcribed as VALUES (not code) with the file:line they come from.

The reference (/root/reference/proj) cannot be built or run in this image (Eigen 3 and the
vendored doctest/CLI11 are missing), so these KATs -- plus the reference's randomized-oracle
properties restated in tests/ -- are what pins the CPU oracle and the GPU kernels.
Run: python tests/golden/make_kats.py   (no dependencies beyond the stdlib)
"""
import json
import math
from pathlib import Path

KATS = {
    "expert_capacity": [
        # (k, f, T, E) -> cap                                  test_core.cpp:8-13, acceptance.cpp:302
        {"k": 1, "f": 1.0, "T": 16384, "E": 2048, "cap": 8, "src": "test_core.cpp:8"},
        {"k": 2, "f": 1.0, "T": 16, "E": 4, "cap": 8, "src": "test_core.cpp:9"},
        {"k": 2, "f": 1.25, "T": 16, "E": 4, "cap": 10, "src": "test_core.cpp:10"},
        {"k": 1, "f": 0.5, "T": 3, "E": 4, "cap": 1, "src": "test_core.cpp:11"},
        {"k": 1, "f": 1.0, "T": 5, "E": 4, "cap": 2, "src": "test_core.cpp:12"},
        {"k": 1, "f": 2.0, "T": 8, "E": 4, "cap": 4, "src": "test_core.cpp:13"},
        {"k": 2, "f": 1.25, "T": 10, "E": 4, "cap": 7, "src": "SPEC.md:58"},
    ],
    "expert_capacity_invalid": [
        {"k": 1, "f": 0.0, "T": 8, "E": 4, "src": "test_core.cpp:14"},
        {"k": 0, "f": 1.0, "T": 8, "E": 4, "src": "test_core.cpp:15"},
    ],
    "resolve_capacity": [
        # kind: 0 fixed, 1 auto, 2 bounded                     test_core.cpp:75-85
        {"kind": 0, "factor": 1.0, "demand": [12, 10, 6, 4], "E": 4, "k": 2, "T": 16, "cap": 8, "src": "test_core.cpp:78"},
        {"kind": 0, "factor": 0.25, "demand": [12, 10, 6, 4], "E": 4, "k": 2, "T": 16, "cap": 2, "src": "test_core.cpp:79"},
        {"kind": 1, "factor": 0.0, "demand": [12, 10, 6, 4], "E": 4, "k": 2, "T": 16, "cap": 12, "src": "test_core.cpp:81"},
        {"kind": 1, "factor": 0.0, "demand": [0, 0, 0, 0], "E": 4, "k": 2, "T": 16, "cap": 1, "src": "test_core.cpp:82"},
        {"kind": 2, "factor": 1.25, "demand": [12, 10, 6, 4], "E": 4, "k": 2, "T": 16, "cap": 10, "src": "test_core.cpp:84"},
        {"kind": 2, "factor": 4.0, "demand": [12, 10, 6, 4], "E": 4, "k": 2, "T": 16, "cap": 12, "src": "test_core.cpp:85"},
        {"kind": 0, "factor": 4.0, "demand": [6, 2], "E": 2, "k": 1, "T": 8, "cap": 16, "src": "SPEC.md:72"},
        {"kind": 1, "factor": 0.0, "demand": [6, 2], "E": 2, "k": 1, "T": 8, "cap": 6, "src": "SPEC.md:73"},
        {"kind": 2, "factor": 1.0, "demand": [6, 2], "E": 2, "k": 1, "T": 8, "cap": 4, "src": "SPEC.md:74"},
    ],
    "capacity_factor_round_trip": {
        # test_core.cpp:18-33: expert_capacity(k, capacity_to_factor(c)) == c
        "k": 2, "T": 16, "E": 8, "fs": [0.5, 1.0, 1.5, 2.0, 4.0], "src": "test_core.cpp:18-33",
    },
    "softmax": [
        # gate_linear on x = 0 -> uniform                      test_gating.cpp:32-35
        {"x": [[0.0, 0.0, 0.0], [0.0, 0.0, 0.0]], "wg": [[0.3, -0.2, 0.9, 0.1], [0.5, 0.5, -1.0, 0.2], [0.7, 0.0, 0.4, -0.6]],
         "probs": [[0.25] * 4, [0.25] * 4], "src": "test_gating.cpp:32-35"},
        # softmax(0, ln 3) = [0.25, 0.75]
        {"x": [[1.0]], "wg": [[0.0, math.log(3.0)]], "probs": [[0.25, 0.75]], "src": "SPEC.md:122"},
    ],
    "topk": [
        {"probs": [[0.1, 0.4, 0.4, 0.1], [0.25, 0.25, 0.25, 0.25]], "k": 2,
         "idxs": [[1, 2], [0, 1]], "gate00": 0.4, "src": "test_gating.cpp:55-65"},
        {"probs": [[0.1, 0.7, 0.2]], "k": 1, "idxs": [[1]], "gate00": 0.7, "src": "SPEC.md:139"},
    ],
    "assign_locations": [
        {"idxs": [0, 0, 0, 1], "gates": [0.9, 0.5, 0.7, 0.3], "cap": 2, "bpr": 0,
         "locations": [0, 1, -1, 0], "src": "test_gating.cpp:67-77"},
        {"idxs": [0, 0, 0, 1], "gates": [0.5, 0.9, 0.7, 0.3], "cap": 2, "bpr": 1,
         "locations": [-1, 0, 1, 0], "src": "test_gating.cpp:79-89"},
        {"idxs": [0, 0, 0], "gates": [0.5, 0.5, 0.5], "cap": 2, "bpr": 1,
         "locations": [0, 1, -1], "src": "test_gating.cpp:91-100"},
        {"idxs": [0, 0, 0], "gates": [0.3, 0.3, 0.3], "cap": 2, "bpr": 0,
         "locations": [0, 1, -1], "src": "SPEC.md:148"},
        {"idxs": [0, 0, 0], "gates": [0.2, 0.5, 0.9], "cap": 2, "bpr": 1,
         "locations": [-1, 1, 0], "src": "SPEC.md:149"},
    ],
    "run_gating": [
        # E=2, T=4, k=1                                        test_gating.cpp:102-115
        {"probs": [[0.9, 0.1], [0.8, 0.2], [0.7, 0.3], [0.2, 0.8]], "k": 1, "blocks": 1,
         "kind": 1, "factor": 0.0, "cap": 3, "drops": 0, "src": "test_gating.cpp:110-111"},
        {"probs": [[0.9, 0.1], [0.8, 0.2], [0.7, 0.3], [0.2, 0.8]], "k": 1, "blocks": 1,
         "kind": 0, "factor": 0.5, "cap": 1, "drops": 2, "src": "test_gating.cpp:112-114"},
        # two blocks of two tokens, all to expert 0            test_gating.cpp:117-136
        {"probs": [[0.9, 0.1], [0.8, 0.2], [0.7, 0.3], [0.6, 0.4]], "k": 1, "blocks": 2,
         "kind": 1, "factor": 0.0, "cap": 2, "locations": [0, 1, 0, 1], "src": "test_gating.cpp:129-135"},
    ],
    "encode": [
        # T=2, M=1, E=2, cap=1, k=1; token0 -> (e1,c0), token1 -> (e0,c0)
        {"x": [[1.0], [2.0]], "E": 2, "cap": 1, "idxs": [1, 0], "locations": [0, 0],
         "z": [[[2.0]], [[1.0]]], "src": "SPEC.md:192"},
    ],
    "expert_ffn": [
        # M=V=1, w1=1, w2=2: x=3 -> 6, x=-3 -> 0            test_parallelism.cpp:82-104
        {"x": [[[3.0], [-3.0]]], "w1": [[[1.0]]], "w2": [[[2.0]]], "y": [[[6.0], [0.0]]],
         "src": "test_parallelism.cpp:82-95"},
        # identity 2x2 weights: relu passthrough
        {"x": [[[-1.0, 5.0]]], "w1": [[[1.0, 0.0], [0.0, 1.0]]],
         "w2": [[[1.0, 0.0], [0.0, 1.0]]], "y": [[[0.0, 5.0]]],
         "src": "test_parallelism.cpp:96-104"},
    ],
    "partition_capacity": {
        # (E=2, C=3, M=4), d=2 -> two chunks of cc=2, tail padded  test_pipeline.cpp:18-37
        "E": 2, "C": 3, "M": 4, "degree": 2, "cc": 2, "src": "test_pipeline.cpp:18-37",
    },
    "flex_all2all": {
        # out[d][e][r*dC+c] == in[r][d*dE+e][c]                test_collectives.cpp:155-181
        "W": 2, "E": 4, "dC": 2, "M": 3, "src": "test_collectives.cpp:155-181",
    },
    "alg1_buckets": [
        {"fs": [1.0, 1.1, 4.0], "members": [[1.0, 1.1], [4.0]], "src": "test_pipeline.cpp:99-107"},
        {"fs": [1.0, 1.4, 1.6], "members": [[1.0, 1.4], [1.6]], "src": "test_pipeline.cpp:108-114"},
    ],
    "alg1_normalization": {
        # optimize(2.0, s0, 10.0); optimize(2.4, s0, 24.0) -> bucket[s0] = 24*2/2.4 = 20
        "f1": 2.0, "t1": 10.0, "f2": 2.4, "t2": 24.0, "bucket": 20.0, "src": "test_pipeline.cpp:116-127",
    },
    "alg1_explore_exploit": {
        # strategy i costs 10 - i: explore the 8 in order, then exploit the last  test_pipeline.cpp:129-147
        "f": 1.0, "steps": 11, "src": "test_pipeline.cpp:129-147",
    },
    "alg1_bucket_sharing": {
        # f=1.0 fully explored with 2dhx4 (index 6) best; f=1.2 exploits it; f=3.0 explores index 0
        "winner": 6, "near_f": 1.2, "far_f": 3.0, "src": "test_pipeline.cpp:149-160",
    },
    "rng": {
        # Rng(123) determinism and range                       test_core.cpp:106-124
        "seed": 123, "n": 1000, "src": "test_core.cpp:106-124",
    },
}

if __name__ == "__main__":
    out = Path(__file__).with_name("reference_kats.json")
    out.write_text(json.dumps(KATS, indent=1))
    print(out)
