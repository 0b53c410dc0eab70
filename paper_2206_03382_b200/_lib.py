"""ctypes binding of libmoe_b200.so (the C ABI declared in include/moe_b200.h).

Loading the library needs no GPU (so symbol checks run on CPU-only hosts); every compute entry
point fails loudly (MoeError) when the CUDA device or the library is missing -- there is no
fallback path.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

_PKG = Path(__file__).resolve().parent
# MOE_LIB_PATH selects an alternative build of the same library (tuning variants); default in-tree.
LIB_PATH = Path(os.environ.get("MOE_LIB_PATH", _PKG / "libmoe_b200.so"))

MOE_OK, MOE_EINVAL, MOE_ECUDA, MOE_ECOMM, MOE_ESTATE, MOE_ENOMEM = range(6)
DTYPE_BF16, DTYPE_F32, DTYPE_F64 = 0, 1, 2
CAP_FIXED, CAP_AUTO, CAP_BOUNDED = 0, 1, 2

PHASES = ["gate", "encode", "gemm_up", "gemm_down", "decode", "decode_bwd", "gemm_dgrad_mask",
          "gemm_dgrad", "gemm_wgrad1", "gemm_wgrad2", "encode_bwd", "a2a_fwd", "a2a_bwd",
          "assign", "relu_fixup", "xfer_dispatch", "xfer_combine", "weight_stats"]

_ERRNAMES = {1: "EINVAL", 2: "ECUDA", 3: "ECOMM", 4: "ESTATE", 5: "ENOMEM"}


class MoeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{_ERRNAMES.get(code, code)}] {msg}")
        self.code = code


class MoeConfig(C.Structure):
    _fields_ = [
        ("world_size", C.c_int64), ("gpus_per_node", C.c_int64), ("global_experts", C.c_int64),
        ("model_dim", C.c_int64), ("hidden_dim", C.c_int64), ("tokens_per_step", C.c_int64),
        ("top_k", C.c_int64), ("capacity_kind", C.c_int32), ("capacity_factor", C.c_double),
        ("bpr", C.c_int32), ("dtype", C.c_int32), ("adaptive", C.c_int32), ("degree", C.c_int32),
        ("a2a_backend", C.c_int32), ("router", C.c_int32), ("parallel", C.c_int32),
        ("a2a_algo", C.c_int32), ("gate_precision", C.c_int32),
    ]


class StepMetrics(C.Structure):
    _fields_ = [
        ("f", C.c_double), ("capacity", C.c_int64), ("a2a_algo", C.c_int32),
        ("degree", C.c_int32), ("seconds", C.c_double), ("comm_bytes", C.c_double),
        ("drop_count", C.c_int64), ("relu_fixups", C.c_int64), ("fused", C.c_int32),
        ("parallel", C.c_int32), ("gate_fixups", C.c_int64), ("simt_gemms", C.c_int64),
    ]


P = C.c_void_p
I32, I64, U64, D = C.c_int32, C.c_int64, C.c_uint64, C.c_double
PI32, PI64, PD, PF = C.POINTER(I32), C.POINTER(I64), C.POINTER(D), C.POINTER(C.c_float)

# name -> (restype, argtypes)
SIGNATURES = {
    "moe_expert_capacity": (I32, [I64, D, I64, I64, PI64]),
    "moe_resolve_capacity": (I32, [I32, D, PI64, I64, I64, I64, PI64]),
    "moe_capacity_to_factor": (I32, [I64, I64, I64, I64, PD]),
    "moe_validate_config": (I32, [C.POINTER(MoeConfig)]),
    "moe_select_parallelism": (I32, [D, I64, I64, D, I64, PI32]),
    "moe_a2a_plan": (I32, [I64, I64, I64, I64, I64, I32, PI64, PI64, PI64]),
    "moe_get_unique_id": (I32, [C.c_char_p]),
    "moe_create": (I32, [C.POINTER(MoeConfig), I32, C.c_char_p, I32, C.POINTER(P)]),
    "moe_destroy": (I32, [P]),
    "moe_last_error": (C.c_char_p, [P]),
    "moe_last_error_global": (C.c_char_p, []),
    "moe_init_params": (I32, [P, U64]),
    "moe_set_router": (I32, [P, P]),
    "moe_set_cosine_router": (I32, [P, P, P, D]),
    "moe_set_capacity_factor": (I32, [P, D]),
    "moe_set_expert": (I32, [P, I64, P, P]),
    "moe_set_expert_slices": (I32, [P, P, P]),
    "moe_forward": (I32, [P, P, P, P]),
    "moe_backward": (I32, [P, P, P, P, P, P]),
    "moe_forward_host": (I32, [P, P, P, P]),
    "moe_backward_host": (I32, [P, P, P, P]),
    "moe_forward_host_async": (I32, [P, P, P, P]),
    "moe_backward_host_async": (I32, [P, P, P, P]),
    "moe_host_sync": (I32, [P]),
    "moe_get_routing": (I32, [P, P, P, P, PI64]),
    "moe_get_metrics": (I32, [P, C.POINTER(StepMetrics)]),
    "moe_get_expert_grads": (I32, [P, P, P]),
    "moe_get_weights_device": (I32, [P, I32, C.POINTER(P)]),
    "moe_weights_updated": (I32, [P]),
    "moe_set_kernel_spans": (I32, [P, I32]),
    "moe_take_kernel_spans": (I32, [P, PD, PI64, I32, PD]),
    "moe_get_expert_grad_slices": (I32, [P, P, P, P]),
    "moe_kernel_launches": (I64, [P]),
    "moe_set_profiling": (I32, [P, I32]),
    "moe_take_profile": (I32, [P, PD, PI64, I32]),
    "moe_op_gating": (I32, [P, I32, P, I64, I64, I64, I64, I64, I32, D, I32, P, P, P, P, PI64,
                            PI64, P]),
    "moe_op_gating_cosine": (I32, [P, I32, P, P, I64, D, I64, I64, I64, I64, I64, I32, D, I32, P, P,
                                   P, P, PI64, PI64, P]),
    "moe_op_encode": (I32, [P, I32, I64, I64, I64, I64, I64, I64, I64, P, P, P, P]),
    "moe_op_decode": (I32, [P, I32, I64, I64, I64, I64, I64, I64, I64, P, P, P, P, P]),
    "moe_op_decode_backward": (I32, [P, P, I32, I64, I64, I64, I64, I64, I64, I64, P, P, P, P, P,
                                     P]),
    "moe_op_encode_backward": (I32, [P, I32, I64, I64, I64, I64, I64, I64, I64, P, P, P, P]),
    "moe_op_expert_ffn": (I32, [P, P, P, P, P, I32, I64, I64, I64, I64, P]),
    "moe_op_expert_ffn_backward": (I32, [P, P, P, P, P, P, P, I32, I64, I64, I64, I64, P]),
    "moe_op_weight_stats": (I32, [P, I64, I64, I64, PF, PF, P, P]),
    "moe_op_gemm": (I32, [I32, I32, I32, P, P, P, P, I64, I64, I64, I64, I64, I64, I64, I64, P]),
    "moe_op_fill_uniform": (I32, [P, I32, I64, U64, U64, D, D, P]),
    "moe_memo_create": (I32, [D, C.POINTER(P)]),
    "moe_memo_destroy": (I32, [P]),
    "moe_memo_get_strategy": (I32, [P, D, PI32]),
    "moe_memo_optimize_strategy": (I32, [P, D, I32, D]),
    "moe_memo_recompute_buckets": (I32, [P, D]),
    "moe_memo_num_buckets": (I32, [P, PI64]),
    "moe_memo_bucket": (I32, [P, I64, PD, PI64, PD, I64, PD]),
    "moe_memo_lookup": (I32, [P, D, I32, PD, PI32]),
}

_lib = None


def lib() -> C.CDLL:
    """Load (once) the in-tree library; raises if it was not built."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise MoeError(MOE_ECUDA, f"{LIB_PATH} missing: run `python -m paper_2206_03382_b200.build`"
                                      " (no CPU fallback exists)")
        l = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib


def check(rc: int, handle=None) -> None:
    if rc != MOE_OK:
        l = lib()
        msg = l.moe_last_error(handle) if handle else l.moe_last_error_global()
        raise MoeError(rc, (msg or b"").decode(errors="replace"))
