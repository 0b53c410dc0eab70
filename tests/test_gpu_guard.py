"""Out-of-bounds write detection without compute-sanitizer (closed on this pool): every output of
the layer and of the sub-operators is placed inside a larger allocation whose guard bands are
filled with a byte pattern; after the call the bands must be untouched and every output still
matches the oracle. Covers the ragged / tail cases where an off-by-one store would land: token
counts that are not multiples of the 64-token gate block, capacities that do not divide into the
pipelining degree, k = 2 with drops, SIMT and tensor-core GEMM shapes.

Also: the same step with programmatic dependent launch on and off (MOE_PDL=0, a fresh process)
must be bit-identical -- an inter-kernel race that PDL's overlap exposes would differ."""
import ctypes as C
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

import oracle
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward
from paper_2206_03382_b200._lib import check, lib
from tests.helpers import layer_inputs

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]
GUARD = 4096  # bytes of guard band on each side
PATTERN = 0xA5


class Guarded:
    """A tensor of `shape` / `dtype` in the middle of a byte buffer with guard bands."""

    def __init__(self, shape, dtype, fill=None):
        n = int(np.prod(shape)) * torch.empty(0, dtype=dtype).element_size()
        self.raw = torch.full((GUARD + n + GUARD,), PATTERN, dtype=torch.uint8, device="cuda")
        self.t = self.raw[GUARD:GUARD + n].view(dtype).view(*shape)
        if fill is not None:
            self.t.copy_(fill)
        self.n = n

    def intact(self) -> bool:
        torch.cuda.synchronize()
        lo, hi = self.raw[:GUARD], self.raw[GUARD + self.n:]
        return bool((lo == PATTERN).all()) and bool((hi == PATTERN).all())


@pytest.mark.parametrize("E,k,f,M,V,T,bpr,dt,degree", [
    (8, 2, 0.75, 256, 512, 1000, True, "bf16", 1),   # ragged token block, drops, BPR
    (6, 1, 1.0, 40, 72, 300, False, "bf16", 1),      # SIMT GEMM shapes
    (8, 1, 1.0, 512, 1024, 4096, False, "bf16", 1),  # tcgen05, certified gate, fused decode
    (4, 2, 1.25, 64, 128, 200, True, "f32", 1),      # fp32 DMMA path
])
def test_layer_outputs_stay_in_bounds(cuda, E, k, f, M, V, T, bpr, dt, degree):
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=k,
                         capacity_factor=f, bpr=bpr, dtype=dt, degree=degree)
    inp = layer_inputs(61, 1, T, M, V, E, dt)
    st = LayerState.init(cfg, 61)
    tdt = cfg.torch_dtype
    x = torch.as_tensor(inp["x"]).to(tdt).cuda()
    dy = torch.as_tensor(inp["dy"]).to(tdt).cuda()
    y = Guarded((T, M), tdt)
    dx = Guarded((T, M), tdt)
    dw1 = Guarded((E, M, V), torch.float32)
    dw2 = Guarded((E, V, M), torch.float32)
    for _ in range(2):  # the second step reuses every internal buffer
        res = forward(st, x, y.t)
        backward(st, res.saved, dy, dx.t, dw1.t, dw2.t)
    assert y.intact() and dx.intact() and dw1.intact() and dw2.intact()
    ref = oracle.layer_step(inp["x"], inp["wg"], inp["w1"], inp["w2"], inp["dy"], 1, k, 0, f, bpr)
    tol = 1e-5 if dt == "f32" else 2e-2
    for name, got in (("y", y.t), ("dx", dx.t), ("dw1", dw1.t), ("dw2", dw2.t)):
        assert oracle.max_rel_diff(got.double().cpu().numpy(), ref[name]) < tol, name
    st.close()


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def test_sub_operators_stay_in_bounds(cuda):
    """Gating (Auto capacity, BPR, probs), encode / decode / decode-backward (+d_gates) /
    encode-backward with a capacity that does not divide into the degree, weight stats."""
    blocks, T, M, E, k, degree = 2, 777, 128, 8, 2, 3
    n = blocks * T
    rs = np.random.RandomState(5)
    x = torch.as_tensor(rs.uniform(-1, 1, (n, M))).to(torch.bfloat16).cuda()
    wg = torch.as_tensor(rs.uniform(-1, 1, (M, E))).cuda()
    idxs = Guarded((n, k), torch.int32)
    gates = Guarded((n, k), torch.float64)
    loc = Guarded((n, k), torch.int32)
    probs = Guarded((n, E), torch.float64)
    cap, drops = C.c_int64(), C.c_int64()
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    check(lib().moe_op_gating(_p(x), 0, _p(wg), blocks, T, M, E, k, 1, 1.0, 1, _p(idxs.t),
                              _p(gates.t), _p(loc.t), _p(probs.t), C.byref(cap), C.byref(drops), st))
    assert idxs.intact() and gates.intact() and loc.intact() and probs.intact()
    cap = cap.value
    cc = -(-cap // degree)
    z = Guarded((blocks, degree, E, cc, M), torch.bfloat16)
    check(lib().moe_op_encode(_p(x), 0, blocks, T, M, E, k, cap, degree, _p(idxs.t), _p(loc.t),
                              _p(z.t), st))
    y = Guarded((n, M), torch.bfloat16)
    check(lib().moe_op_decode(_p(z.t), 0, blocks, T, M, E, k, cap, degree, _p(idxs.t), _p(loc.t),
                              _p(gates.t), _p(y.t), st))
    dz = Guarded((blocks, degree, E, cc, M), torch.bfloat16)
    dg = Guarded((n, k), torch.float64)
    check(lib().moe_op_decode_backward(_p(x), _p(z.t), 0, blocks, T, M, E, k, cap, degree,
                                       _p(idxs.t), _p(loc.t), _p(gates.t), _p(dz.t), _p(dg.t), st))
    dx = Guarded((n, M), torch.bfloat16)
    check(lib().moe_op_encode_backward(_p(dz.t), 0, blocks, T, M, E, k, cap, degree, _p(idxs.t),
                                       _p(loc.t), _p(dx.t), st))
    for g in (z, y, dz, dg, dx):
        assert g.intact()
    # the values themselves: encode byte-exact against the oracle's layout
    xe = x.double().cpu().numpy()
    oz = oracle.encode(xe, blocks, E, k, cap, idxs.t.cpu().numpy().astype(np.int64),
                       loc.t.cpu().numpy().astype(np.int64))
    want = np.stack([oracle.partition_capacity(oz[b], degree) for b in range(blocks)])
    assert np.array_equal(z.t.double().cpu().numpy(), want)
    w1 = (torch.rand(3, 192, 320, device="cuda", dtype=torch.float64) - 0.5).to(torch.bfloat16)
    cn = Guarded((3, 320), torch.float32)
    blk = Guarded((3, 5), torch.float32)
    w1t = Guarded((3, 320, 192), torch.bfloat16)
    check(lib().moe_op_weight_stats(_p(w1), 3, 192, 320, C.cast(_p(cn.t), C.POINTER(C.c_float)),
                                    C.cast(_p(blk.t), C.POINTER(C.c_float)), _p(w1t.t), st))
    assert cn.intact() and blk.intact() and w1t.intact()
    assert torch.equal(w1t.t, w1.transpose(1, 2).contiguous())


_PDL_SCRIPT = r"""
import hashlib, sys, torch
sys.path.insert(0, {root!r})
from paper_2206_03382_b200 import LayerState, MoELayerConfig, backward, forward
from tests.helpers import layer_inputs
E, k, f, M, V, T = 16, 1, 1.0, 512, 1024, 4096
for bpr, kk in ((False, 1), (True, 2)):
    cfg = MoELayerConfig(global_experts=E, model_dim=M, hidden_dim=V, tokens_per_step=T, top_k=kk,
                         capacity_factor=1.25, bpr=bpr, dtype="bf16")
    inp = layer_inputs(7, 1, T, M, V, E, "bf16")
    st = LayerState.init(cfg, 7)
    x = torch.as_tensor(inp["x"]).to(torch.bfloat16).cuda()
    dy = torch.as_tensor(inp["dy"]).to(torch.bfloat16).cuda()
    res = forward(st, x)
    g = backward(st, res.saved, dy)
    torch.cuda.synchronize()
    h = hashlib.sha256()
    for t in (res.y, g.dx, g.dw1, g.dw2):
        h.update(t.contiguous().view(torch.uint8).cpu().numpy().tobytes())
    print(h.hexdigest())
"""


def test_pdl_on_off_bit_identical(cuda):
    """Programmatic dependent launch overlaps each kernel's prologue with its predecessor's tail;
    a missing dependency wait would make results timing-dependent. Same digests with it off."""
    out = {}
    for pdl in ("1", "0"):
        env = dict(os.environ, MOE_PDL=pdl)
        r = subprocess.run([sys.executable, "-c", _PDL_SCRIPT.format(root=str(ROOT))], env=env,
                           capture_output=True, text=True, timeout=600, cwd=ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        out[pdl] = r.stdout.split()
    assert len(out["1"]) == 2 and out["1"] == out["0"]
