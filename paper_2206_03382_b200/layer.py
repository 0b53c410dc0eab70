"""Python mirror of the reference layer API (moe_layer.hpp) over the C ABI.

    state = LayerState.init(MoELayerConfig(...), seed=402)     # LayerState::init
    res = forward(state, x)                                    # forward(state, x)
    grads = backward(state, res.saved, dy)                     # backward(state, saved, dy)

x / dy are this rank's (T, M) token block as torch CUDA tensors in the layer dtype. All work
runs in libmoe_b200.so (sm_100a kernels + NCCL); there is no Python or CPU compute path.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import torch

from . import _lib
from ._lib import MoeConfig, StepMetrics, check, lib

_DT = {"bf16": _lib.DTYPE_BF16, "f32": _lib.DTYPE_F32}
_TORCH_DT = {"bf16": torch.bfloat16, "f32": torch.float32}
_CAP = {"fixed": _lib.CAP_FIXED, "auto": _lib.CAP_AUTO, "bounded": _lib.CAP_BOUNDED}


@dataclass
class MoELayerConfig:
    """MoELayerConfig + Dims (moe_layer.hpp:22-29, core.hpp:32-56). E >= W: per-rank placement
    (E/W experts per rank); E < W: sharded placement (W = E*s, rank r serves expert r/s)."""
    world_size: int = 1
    gpus_per_node: int = 1
    global_experts: int = 1
    model_dim: int = 1
    hidden_dim: int = 1
    tokens_per_step: int = 1
    top_k: int = 1
    capacity: str = "fixed"
    capacity_factor: float = 1.0
    bpr: bool = False
    dtype: str = "bf16"
    adaptive: bool = False
    degree: int = 1
    a2a_backend: str = "peer"   # "peer" (copy engines over NVLink) or "nccl"
    router: str = "linear"      # RouterKind (moe_layer.hpp:10): "linear" or "cosine"
    parallel: str = "p1"        # ParallelControl (sharded placement): "p1", "p2" or "adaptive"
    a2a_algo: str = "linear"    # StrategyControl::fixed.algo: "linear" or "2dh"
    gate_precision: str = "auto"  # "auto" (certified tensor-core gate where it applies) or "fp64"

    def to_c(self) -> MoeConfig:
        return MoeConfig(self.world_size, self.gpus_per_node, self.global_experts, self.model_dim,
                         self.hidden_dim, self.tokens_per_step, self.top_k, _CAP[self.capacity],
                         float(self.capacity_factor), int(self.bpr), _DT[self.dtype],
                         int(self.adaptive), int(self.degree),
                         {"peer": 0, "nccl": 1}[self.a2a_backend],
                         {"linear": 0, "cosine": 1}[self.router],
                         {"p1": 0, "p2": 1, "adaptive": 2}[self.parallel],
                         {"linear": 0, "2dh": 1}[self.a2a_algo],
                         {"auto": 0, "fp64": 1}[self.gate_precision])

    @property
    def local_experts(self) -> int:
        """Experts this rank computes: E/W, or 1 under sharded placement."""
        return max(1, self.global_experts // self.world_size)

    @property
    def n_sharded(self) -> int:
        """s of RanksPerExpert{s} (W = E*s); 1 under per-rank placement."""
        return self.world_size // self.global_experts if self.global_experts < self.world_size else 1

    @property
    def torch_dtype(self) -> torch.dtype:
        return _TORCH_DT[self.dtype]

    def validate(self) -> None:
        c = self.to_c()
        check(lib().moe_validate_config(C.byref(c)))


@dataclass
class StepMetricsPy:
    f: float
    capacity: int
    a2a_algo: str
    degree: int
    seconds: float
    comm_bytes: float
    drop_count: int
    relu_fixups: int = 0
    fused: int = 0  # MOE_FUSED_DECODE (1) | MOE_FUSED_COMBINE (2)
    parallel: str = "p1"  # StepMetrics::parallel
    gate_fixups: int = 0  # certified gate: tokens re-decided in fp64 since the last read
    simt_gemms: int = 0   # bf16 GEMM launches that fell back to the SIMT kernel (shape cliff)


@dataclass
class SavedForward:
    """Handle-owned saved tensors of the last forward (SavedForward, moe_layer.hpp:56-66)."""
    step: int


@dataclass
class ForwardResult:
    y: torch.Tensor
    saved: SavedForward
    state: "LayerState" = field(repr=False, default=None)

    @property
    def metrics(self) -> StepMetricsPy:
        return self.state.metrics()


@dataclass
class LayerGrads:
    dx: torch.Tensor
    dw1: torch.Tensor  # (E/W, M, V) fp32, local experts
    dw2: torch.Tensor  # (E/W, V, M) fp32


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _stream(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


class LayerState:
    """One rank's layer (LayerState, moe_layer.hpp:33-44) backed by a moe_handle."""

    def __init__(self, config: MoELayerConfig, rank: int = 0, device: int = 0,
                 nccl_id: bytes | None = None):
        self.config = config
        self.rank = rank
        self.device = torch.device("cuda", device)
        self._h = C.c_void_p()
        c = config.to_c()
        check(lib().moe_create(C.byref(c), rank, nccl_id, device, C.byref(self._h)))
        self._step = 0

    @staticmethod
    def unique_id() -> bytes:
        buf = C.create_string_buffer(128)
        check(lib().moe_get_unique_id(buf))
        return buf.raw

    @classmethod
    def init(cls, config: MoELayerConfig, seed: int, rank: int = 0, device: int = 0,
             nccl_id: bytes | None = None) -> "LayerState":
        """LayerState::init (moe_layer.cpp:144-163) with the Rng(seed) draw order."""
        s = cls(config, rank, device, nccl_id)
        check(lib().moe_init_params(s._h, C.c_uint64(seed)), s._h)
        return s

    def close(self) -> None:
        if self._h:
            lib().moe_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- parameters
    def set_router(self, wg) -> None:
        import numpy as np
        a = np.ascontiguousarray(wg, np.float64)
        check(lib().moe_set_router(self._h, a.ctypes.data_as(C.c_void_p)), self._h)

    def set_capacity_factor(self, f: float) -> None:
        """FixedCapacity{f} from the next forward on (collective for W > 1)."""
        check(lib().moe_set_capacity_factor(self._h, float(f)), self._h)

    def set_cosine_router(self, proj, experts, temperature: float = 1.0) -> None:
        """RouterParams cosine_proj (M, 256), cosine_experts (E, 256), temperature."""
        import numpy as np
        a = np.ascontiguousarray(proj, np.float64)
        b = np.ascontiguousarray(experts, np.float64)
        check(lib().moe_set_cosine_router(self._h, a.ctypes.data_as(C.c_void_p),
                                          b.ctypes.data_as(C.c_void_p), float(temperature)), self._h)

    def set_expert(self, local_e: int, w1, w2) -> None:
        import numpy as np
        a = np.ascontiguousarray(w1, np.float64)
        b = np.ascontiguousarray(w2, np.float64)
        check(lib().moe_set_expert(self._h, local_e, a.ctypes.data_as(C.c_void_p),
                                   b.ctypes.data_as(C.c_void_p)), self._h)

    def set_expert_slices(self, w1_slices, w2_slices) -> None:
        import numpy as np
        a = np.ascontiguousarray(w1_slices, np.float64)
        b = np.ascontiguousarray(w2_slices, np.float64)
        check(lib().moe_set_expert_slices(self._h, a.ctypes.data_as(C.c_void_p),
                                          b.ctypes.data_as(C.c_void_p)), self._h)

    def weights(self):
        """Device views (E/W, M, V) / (E/W, V, M) of the resident local expert weights. Writable:
        fetching them marks the derived weight state stale; after writing through views kept
        from an earlier call, call weights_updated() before the next forward."""
        cfg = self.config
        out = []
        for which, shape in ((1, (cfg.local_experts, cfg.model_dim, cfg.hidden_dim)),
                             (2, (cfg.local_experts, cfg.hidden_dim, cfg.model_dim))):
            p = C.c_void_p()
            check(lib().moe_get_weights_device(self._h, which, C.byref(p)), self._h)
            n = shape[0] * shape[1] * shape[2]
            esz = 2 if cfg.dtype == "bf16" else 4
            out.append(_from_ptr(p.value, n * esz, cfg.torch_dtype, shape, self.device))
        return out

    def expert_grads(self):
        """Host fp32 copies of the last backward's local expert gradients (moe_get_expert_grads),
        wherever backward wrote them; MoeError before any backward."""
        import numpy as np
        cfg = self.config
        n_e = cfg.local_experts
        w1 = np.empty((n_e, cfg.model_dim, cfg.hidden_dim), np.float32)
        w2 = np.empty((n_e, cfg.hidden_dim, cfg.model_dim), np.float32)
        check(lib().moe_get_expert_grads(self._h, w1.ctypes.data_as(C.c_void_p),
                                         w2.ctypes.data_as(C.c_void_p)), self._h)
        return w1, w2

    def weights_updated(self) -> None:
        """The resident weights were changed in place (moe_weights_updated)."""
        check(lib().moe_weights_updated(self._h), self._h)

    # -- results
    def routing(self):
        import numpy as np
        cfg = self.config
        n = cfg.tokens_per_step * cfg.top_k
        idxs = np.empty(n, np.int32)
        loc = np.empty(n, np.int32)
        gates = np.empty(n, np.float64)
        cap = C.c_int64()
        check(lib().moe_get_routing(self._h, idxs.ctypes.data_as(C.c_void_p),
                                    loc.ctypes.data_as(C.c_void_p),
                                    gates.ctypes.data_as(C.c_void_p), C.byref(cap)), self._h)
        k = cfg.top_k
        return idxs.reshape(-1, k), loc.reshape(-1, k), gates.reshape(-1, k), cap.value

    def metrics(self) -> StepMetricsPy:
        m = StepMetrics()
        check(lib().moe_get_metrics(self._h, C.byref(m)), self._h)
        return StepMetricsPy(m.f, m.capacity, "linear" if m.a2a_algo == 0 else "2dh", m.degree,
                             m.seconds, m.comm_bytes, m.drop_count, m.relu_fixups, m.fused,
                             "p2" if m.parallel == 1 else "p1", m.gate_fixups, m.simt_gemms)

    def grad_slices(self):
        """reduce_scatter_grads_p1: this rank's slice of every expert's dW1 / dW2 (fp32 device),
        shapes (E, M, V/W) and (E, V/W, M); under sharded placement the summed slice r%s of expert
        r/s, shapes (1, M, V/s) and (1, V/s, M). Collective across ranks."""
        cfg = self.config
        s = cfg.n_sharded
        ne = 1 if s > 1 else cfg.global_experts
        h = cfg.hidden_dim // (s if s > 1 else cfg.world_size)
        w1s = torch.empty(ne, cfg.model_dim, h, dtype=torch.float32, device=self.device)
        w2s = torch.empty(ne, h, cfg.model_dim, dtype=torch.float32, device=self.device)
        check(lib().moe_get_expert_grad_slices(self._h, _ptr(w1s), _ptr(w2s), _stream(self.device)),
              self._h)
        return w1s, w2s

    def kernel_launches(self) -> int:
        return int(lib().moe_kernel_launches(self._h))

    def set_profiling(self, on: bool) -> None:
        check(lib().moe_set_profiling(self._h, int(on)), self._h)

    def take_profile(self) -> dict:
        """{phase: (total ms, intervals)} since the last call (measured timeline)."""
        import numpy as np
        n = len(_lib.PHASES)
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.int64)
        check(lib().moe_take_profile(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                     cnt.ctypes.data_as(C.POINTER(C.c_int64)), n), self._h)
        return {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(_lib.PHASES)}

    def set_kernel_spans(self, on: bool) -> None:
        check(lib().moe_set_kernel_spans(self._h, int(on)), self._h)

    def take_kernel_spans(self) -> dict:
        """{phase: (summed GEMM kernel span ms, launches)} from the device clock (no events)."""
        import numpy as np
        n = len(_lib.PHASES)
        ms = np.zeros(n, np.float64)
        cnt = np.zeros(n, np.int64)
        mhz = C.c_double(0.0)
        check(lib().moe_take_kernel_spans(self._h, ms.ctypes.data_as(C.POINTER(C.c_double)),
                                          cnt.ctypes.data_as(C.POINTER(C.c_int64)), n,
                                          C.byref(mhz)), self._h)
        out = {p: (float(ms[i]), int(cnt[i])) for i, p in enumerate(_lib.PHASES)}
        out["_sm_mhz"] = (float(mhz.value), 0)
        return out

    @property
    def handle(self):
        return self._h


def _from_ptr(ptr: int, nbytes: int, dtype, shape, device):
    """Zero-copy torch view of handle-owned device memory (lifetime bound to the handle)."""
    class _Holder:
        __cuda_array_interface__ = {
            "shape": (nbytes,), "typestr": "|u1", "data": (ptr, False), "version": 3,
        }
    raw = torch.as_tensor(_Holder(), device=device)
    return raw.view(dtype).view(*shape)


def forward(state: LayerState, x: torch.Tensor, y: torch.Tensor | None = None) -> ForwardResult:
    """forward(state, x) (moe_layer.cpp:171-244) for this rank's (T, M) block."""
    cfg = state.config
    if x.shape != (cfg.tokens_per_step, cfg.model_dim) or x.dtype != cfg.torch_dtype:
        raise _lib.MoeError(_lib.MOE_EINVAL, "forward: expected (T, M) input in the layer dtype")
    if not x.is_cuda or not x.is_contiguous():
        raise _lib.MoeError(_lib.MOE_EINVAL, "forward: x must be a contiguous CUDA tensor")
    if y is None:
        y = torch.empty_like(x)
    check(lib().moe_forward(state.handle, _ptr(x), _ptr(y), _stream(x.device)), state.handle)
    state._step += 1
    return ForwardResult(y=y, saved=SavedForward(step=state._step), state=state)


def backward(state: LayerState, saved: SavedForward, dy: torch.Tensor,
             dx: torch.Tensor | None = None, dw1: torch.Tensor | None = None,
             dw2: torch.Tensor | None = None) -> LayerGrads:
    """backward(state, saved, dy) (moe_layer.cpp:246-319): routing/gates frozen to the plan."""
    cfg = state.config
    if saved.step != state._step:
        raise _lib.MoeError(_lib.MOE_ESTATE, "backward: saved forward is stale")
    if dy.shape != (cfg.tokens_per_step, cfg.model_dim) or dy.dtype != cfg.torch_dtype:
        raise _lib.MoeError(_lib.MOE_EINVAL, "backward: expected (T, M) gradient in the layer dtype")
    dev = dy.device
    if dx is None:
        dx = torch.empty_like(dy)
    nE, M, V = cfg.local_experts, cfg.model_dim, cfg.hidden_dim
    if dw1 is None:
        dw1 = torch.empty(nE, M, V, device=dev, dtype=torch.float32)
    if dw2 is None:
        dw2 = torch.empty(nE, V, M, device=dev, dtype=torch.float32)
    check(lib().moe_backward(state.handle, _ptr(dy), _ptr(dx), _ptr(dw1), _ptr(dw2),
                             _stream(dev)), state.handle)
    return LayerGrads(dx=dx, dw1=dw1, dw2=dw2)


def forward_host(state: LayerState, x_host: torch.Tensor, y_host: torch.Tensor) -> None:
    """forward with host (pinned) buffers: H2D + forward + D2H inside the call."""
    check(lib().moe_forward_host(state.handle, _ptr(x_host), _ptr(y_host),
                                 _stream(state.device)), state.handle)
    state._step += 1


def backward_host(state: LayerState, dy_host: torch.Tensor, dx_host: torch.Tensor) -> None:
    check(lib().moe_backward_host(state.handle, _ptr(dy_host), _ptr(dx_host),
                                  _stream(state.device)), state.handle)


def forward_host_async(state: LayerState, x_host: torch.Tensor, y_host: torch.Tensor) -> None:
    """Pipelined forward on pinned host buffers: returns after enqueueing; the upload / download
    overlap neighbouring steps. y_host is valid after host_sync(state)."""
    state._step += 1
    check(lib().moe_forward_host_async(state.handle, _ptr(x_host), _ptr(y_host),
                                       _stream(state.device)), state.handle)


def backward_host_async(state: LayerState, dy_host: torch.Tensor, dx_host: torch.Tensor) -> None:
    check(lib().moe_backward_host_async(state.handle, _ptr(dy_host), _ptr(dx_host),
                                        _stream(state.device)), state.handle)


def host_sync(state: LayerState) -> None:
    """Wait for every download enqueued by the *_host_async calls."""
    check(lib().moe_host_sync(state.handle), state.handle)
