"""tcgen05 grouped GEMM (all five expert-FFN kinds) against a plain PyTorch fp32 reference."""
import ctypes as C

import pytest
import torch

from paper_2206_03382_b200._lib import lib, check, DTYPE_BF16, DTYPE_F32

pytestmark = pytest.mark.gpu


def _p(t):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def run_gemm(kind, dtype, use_tc, A, B, D, aux, G, S, seg_rows, seg_base, N, K, Mo, nseg):
    check(lib().moe_op_gemm(kind, dtype, use_tc, _p(A), _p(B), _p(D), _p(aux), G, S, seg_rows,
                            seg_base, N, K, Mo, nseg, None))
    torch.cuda.synchronize()


def rel(a, b):
    a = a.double(); b = b.double()
    return ((a - b).abs().max() / max(a.abs().max().item(), b.abs().max().item(), 1e-300)).item()


@pytest.mark.parametrize("use_tc", [1, 0])
@pytest.mark.parametrize("G,S,seg_rows,M,V", [(2, 1, 256, 256, 512), (3, 2, 200, 512, 768),
                                              (1, 1, 1024, 1024, 4096)])
def test_row_m_kinds(cuda, use_tc, G, S, seg_rows, M, V):
    torch.manual_seed(0)
    nseg = S * G
    bf = torch.bfloat16
    X = torch.randn(nseg, seg_rows, M, device=cuda).to(bf)
    W1 = (torch.randn(G, M, V, device=cuda) / M ** 0.5).to(bf)
    W2 = (torch.randn(G, V, M, device=cuda) / V ** 0.5).to(bf)
    # segment (s, g) at index s*G + g
    Xg = X.view(S, G, seg_rows, M).permute(1, 0, 2, 3).reshape(G, S * seg_rows, M).float()
    act = torch.empty(nseg, seg_rows, V, device=cuda, dtype=bf)
    run_gemm(0, DTYPE_BF16, use_tc, X, W1, act, None, G, S, seg_rows, 0, V, M, 0, nseg)
    ref_act = torch.relu(torch.bmm(Xg, W1.float()))
    got_act = act.view(S, G, seg_rows, V).permute(1, 0, 2, 3).reshape(G, S * seg_rows, V)
    assert rel(got_act, ref_act) < 1e-2
    Y = torch.empty(nseg, seg_rows, M, device=cuda, dtype=bf)
    run_gemm(1, DTYPE_BF16, use_tc, act, W2, Y, None, G, S, seg_rows, 0, M, V, 0, nseg)
    ref_y = torch.bmm(got_act.float(), W2.float())
    got_y = Y.view(S, G, seg_rows, M).permute(1, 0, 2, 3).reshape(G, S * seg_rows, M)
    assert rel(got_y, ref_y) < 1e-2
    # dgrad with mask: dh = (dY W2^T) * [act > 0] -- via moe_op_expert_ffn_backward's path below;
    # here the SIMT path (reads act) and, for tcgen05, an explicit bitmask built from act.
    dY = torch.randn(nseg, seg_rows, M, device=cuda).to(bf)
    dYg = dY.view(S, G, seg_rows, M).permute(1, 0, 2, 3).reshape(G, S * seg_rows, M).float()
    dh = torch.empty(nseg, seg_rows, V, device=cuda, dtype=bf)
    run_gemm(2, DTYPE_BF16, use_tc, dY, W2, dh, act, G, S, seg_rows, 0, V, M, 0, nseg)
    ref_dh = torch.bmm(dYg, W2.float().transpose(1, 2)) * (got_act.float() > 0)
    got_dh = dh.view(S, G, seg_rows, V).permute(1, 0, 2, 3).reshape(G, S * seg_rows, V)
    assert rel(got_dh, ref_dh) < 1e-2
    dX = torch.empty(nseg, seg_rows, M, device=cuda, dtype=bf)
    run_gemm(3, DTYPE_BF16, use_tc, dh, W1, dX, None, G, S, seg_rows, 0, M, V, 0, nseg)
    ref_dx = torch.bmm(got_dh.float(), W1.float().transpose(1, 2))
    got_dx = dX.view(S, G, seg_rows, M).permute(1, 0, 2, 3).reshape(G, S * seg_rows, M)
    assert rel(got_dx, ref_dx) < 1e-2
    # wgrad: dW1 = X^T dh over all rows of all segments; dW2 = act^T dY
    dW1 = torch.empty(G, M, V, device=cuda, dtype=torch.float32)
    run_gemm(4, DTYPE_BF16, use_tc, X, dh, dW1, None, G, S, seg_rows, 0, V, 0, M, nseg)
    ref_dw1 = torch.bmm(Xg.transpose(1, 2), got_dh.float())
    assert rel(dW1, ref_dw1) < 1e-2
    dW2 = torch.empty(G, V, M, device=cuda, dtype=torch.float32)
    run_gemm(4, DTYPE_BF16, use_tc, act, dY, dW2, None, G, S, seg_rows, 0, M, 0, V, nseg)
    ref_dw2 = torch.bmm(got_act.float().transpose(1, 2), dYg)
    assert rel(dW2, ref_dw2) < 1e-2


def test_seg_base_and_fp32(cuda):
    """seg_base selects a chunk of segments; the fp32 SIMT path meets 1e-5."""
    torch.manual_seed(1)
    G, S, rows, M, V = 2, 2, 64, 128, 256
    nseg_total = 2 * S * G
    X = torch.randn(nseg_total, rows, M, device=cuda)
    W1 = torch.randn(G, M, V, device=cuda) / M ** 0.5
    act = torch.zeros(nseg_total, rows, V, device=cuda)
    run_gemm(0, DTYPE_F32, 0, X, W1, act, None, G, S, rows, S, V, M, 0, nseg_total)
    for s in range(S):
        for g in range(G):
            seg = (S + s) * G + g
            ref = torch.relu(X[seg].double() @ W1[g].double())
            assert rel(act[seg], ref) < 1e-5
            assert act[s * G + g].abs().max().item() == 0.0  # untouched chunk
