"""Grouped tcgen05 GEMM (gemm_sm100.cu) against a plain PyTorch fp32 reference of the
same op on the same bf16 operands.  Covers every mode / operand-major / epilogue the
MoE layer uses (expert FFN fwd, dgrad, wgrad; reference nn.cpp:22-121,
parallel_linear.cpp:8-40).  Tolerance: bf16 output rounding -> rel-L2 <= 1e-2."""
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def _gelu(x):
    return 0.5 * x * (1.0 + torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3)))


def _gelu_grad(x):
    t = torch.tanh(0.7978845608028654 * (x + 0.044715 * x ** 3))
    return 0.5 * (1 + t) + 0.5 * x * (1 - t * t) * 0.7978845608028654 * (1 + 3 * 0.044715 * x * x)


def _rel(a, b):
    a = a.double().flatten()
    b = b.double().flatten()
    return float((a - b).norm() / max(b.norm(), 1e-30))


def _segs(rows):
    off = [0]
    for r in rows:
        off.append(off[-1] + r)
    return torch.tensor(off, dtype=torch.int32, device="cuda")


@pytest.mark.parametrize("rows,N,K", [([128], 256, 64), ([256, 0, 384], 512, 192),
                                      ([1024, 896, 1152, 128], 1024, 1024)])
def test_rows_bmn_bias_gelu(rows, N, K):
    import paper_2303_06318_b200 as ted
    torch.manual_seed(0)
    G, R = len(rows), sum(rows)
    A = torch.randn(R, K, device="cuda").bfloat16()
    B = (torch.randn(G, K, N, device="cuda") / K ** 0.5).bfloat16()
    bias = torch.randn(G, N, device="cuda").bfloat16()
    Z = torch.empty(R, N, device="cuda", dtype=torch.bfloat16)
    H = torch.empty_like(Z)
    seg = _segs(rows)
    ted.grouped_gemm(ted.GEMM_ROWS, ted.EPI_BIAS_GELU, G, 0, N, K, seg, R, A, K, False, B, N,
                     K * N, True, Z, N, bias=bias, bias_group_stride=N, aux=H, ld_aux=N)
    torch.cuda.synchronize()
    off = seg.tolist()
    for g in range(G):
        if rows[g] == 0:
            continue
        ref = A[off[g]:off[g + 1]].float() @ B[g].float() + bias[g].float()
        assert _rel(Z[off[g]:off[g + 1]].float(), ref) < 1e-2
        assert _rel(H[off[g]:off[g + 1]].float(), _gelu(ref)) < 1e-2


@pytest.mark.parametrize("rows,N,K", [([256, 128], 256, 256), ([512, 384, 0, 640], 768, 512)])
def test_rows_bk_store_and_bias(rows, N, K):
    import paper_2303_06318_b200 as ted
    torch.manual_seed(1)
    G, R = len(rows), sum(rows)
    A = torch.randn(R, K, device="cuda").bfloat16()
    Bt = (torch.randn(G, N, K, device="cuda") / K ** 0.5).bfloat16()  # [N][K] K-major
    C = torch.empty(R, N, device="cuda", dtype=torch.bfloat16)
    seg = _segs(rows)
    ted.grouped_gemm(ted.GEMM_ROWS, ted.EPI_STORE, G, 0, N, K, seg, R, A, K, False, Bt, K,
                     N * K, False, C, N)
    torch.cuda.synchronize()
    off = seg.tolist()
    for g in range(G):
        if rows[g]:
            ref = A[off[g]:off[g + 1]].float() @ Bt[g].float().T
            assert _rel(C[off[g]:off[g + 1]].float(), ref) < 1e-2
    # bias epilogue with a null bias == store
    C2 = torch.empty_like(C)
    ted.grouped_gemm(ted.GEMM_ROWS, ted.EPI_BIAS, G, 0, N, K, seg, R, A, K, False, Bt, K, N * K,
                     False, C2, N)
    torch.cuda.synchronize()
    assert torch.equal(C2, C)


def test_rows_dgelu_in_place():
    import paper_2303_06318_b200 as ted
    torch.manual_seed(2)
    rows, N, K = [384, 256], 512, 256
    G, R = len(rows), sum(rows)
    A = torch.randn(R, K, device="cuda").bfloat16()
    Bt = (torch.randn(G, N, K, device="cuda") / K ** 0.5).bfloat16()
    Z = torch.randn(R, N, device="cuda").bfloat16()
    Z0 = Z.clone()
    seg = _segs(rows)
    ted.grouped_gemm(ted.GEMM_ROWS, ted.EPI_DGELU, G, 0, N, K, seg, R, A, K, False, Bt, K, N * K,
                     False, Z, N, aux=Z, ld_aux=N)
    torch.cuda.synchronize()
    off = seg.tolist()
    for g in range(G):
        ref = (A[off[g]:off[g + 1]].float() @ Bt[g].float().T) * _gelu_grad(
            Z0[off[g]:off[g + 1]].float())
        assert _rel(Z[off[g]:off[g + 1]].float(), ref) < 1e-2


@pytest.mark.parametrize("rows,M,N", [([128], 128, 256), ([256, 0, 384], 256, 512),
                                      ([2048, 1920, 2176], 1024, 1024), ([640, 128], 512, 768)])
def test_kdim_wgrad(rows, M, N):
    """M % 256 == 0 runs the CTA-pair (cta_group::2) kernel, M = 128 the single-CTA one."""
    import paper_2303_06318_b200 as ted
    torch.manual_seed(3)
    G, R = len(rows), sum(rows)
    A = torch.randn(R, M, device="cuda").bfloat16()   # X   [rows][M]  (MN-major A)
    B = torch.randn(R, N, device="cuda").bfloat16()   # dZ  [rows][N]  (MN-major B)
    C = torch.full((G, M, N), 7.0, device="cuda", dtype=torch.bfloat16)
    seg = _segs(rows)
    ted.grouped_gemm(ted.GEMM_KDIM, ted.EPI_STORE, G, M, N, 0, seg, R, A, M, True, B, N, 0, True,
                     C, N, c_group_stride=M * N)
    torch.cuda.synchronize()
    off = seg.tolist()
    for g in range(G):
        if rows[g] == 0:
            assert torch.count_nonzero(C[g]) == 0  # empty expert -> zero gradient
            continue
        ref = A[off[g]:off[g + 1]].float().T @ B[off[g]:off[g + 1]].float()
        assert _rel(C[g].float(), ref) < 1e-2


def test_config_errors_are_status_2():
    import paper_2303_06318_b200 as ted
    seg = _segs([128])
    A = torch.zeros(128, 64, device="cuda", dtype=torch.bfloat16)
    with pytest.raises(ted.InvalidConfigError):
        ted.grouped_gemm(ted.GEMM_ROWS, 0, 1, 0, 100, 64, seg, 128, A, 64, False, A, 64, 0, False,
                         A, 100)
