"""B200-native Tutel-style MoE layer (arXiv 2206.03382) -- sm_100a kernels behind a C ABI.

Public surface mirrors the reference layer API (moe_layer.hpp): MoELayerConfig, LayerState,
forward, backward; sub-operators in .ops; the raw C ABI in include/moe_b200.h.
"""
from ._lib import MoeError, lib  # noqa: F401
from .layer import (ForwardResult, LayerGrads, LayerState, MoELayerConfig,  # noqa: F401
                    SavedForward, backward, backward_host, forward, forward_host)

__all__ = ["MoELayerConfig", "LayerState", "forward", "backward", "forward_host",
           "backward_host", "ForwardResult", "LayerGrads", "SavedForward", "MoeError", "lib"]
