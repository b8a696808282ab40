"""Numerics of the tcgen05 3xTF32 GEMM through the local_gemm seam
(kernels.hpp:81-89 semantics) against an fp64 PyTorch reference.

Tolerance: relative Frobenius error <= 1e-5 (the reference's fp32 bar,
harness.hpp:114-120); 3xTF32 lands near 1e-7 at these sizes.
"""
import pytest

pytestmark = pytest.mark.gpu

TOL = 1e-5


@pytest.fixture(params=[0, 1], ids=["tf32x3", "mixed"])
def mode(request, monkeypatch):
    """Split-product mode: 0 = 3xTF32, 1 = TF32 + 2xBF16."""
    monkeypatch.setenv("DM_GEMM_MODE", str(request.param))
    return request.param


def _relfro(got, want):
    import torch
    d = (got.double() - want).norm()
    n = want.norm()
    return float(d / n) if n > 0 else float(d)


def _run(cuda, m, n, k, ta, tb, alpha, beta, cg, seed=0):
    import torch
    from paper_1604_01416_b200 import local_gemm
    g = torch.Generator(device="cpu").manual_seed(seed)
    A = (torch.rand((k, m) if ta else (m, k), generator=g) * 2 - 1).to(cuda)
    B = (torch.rand((n, k) if tb else (k, n), generator=g) * 2 - 1).to(cuda)
    C0 = (torch.rand((m, n), generator=g) * 2 - 1).to(cuda)
    C = C0.clone()
    local_gemm(alpha, A, ta, B, tb, beta, C, cta_group=cg)
    torch.cuda.synchronize()
    opA = A.double().T if ta else A.double()
    opB = B.double().T if tb else B.double()
    want = alpha * (opA @ opB)
    if beta != 0.0:
        want = want + beta * C0.double()
    return _relfro(C, want)


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("m,n,k", [(128, 128, 32), (256, 256, 64), (300, 200, 100), (3, 5, 7),
                                   (1024, 1024, 1024), (1000, 1500, 777)])
def test_shapes(cuda, mode, cg, m, n, k):
    assert _run(cuda, m, n, k, False, False, 1.0, 0.0, cg) <= TOL


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("ta,tb", [(False, False), (True, False), (False, True), (True, True)])
def test_transposes_alpha_beta(cuda, mode, cg, ta, tb):
    assert _run(cuda, 520, 390, 260, ta, tb, 1.5, -0.5, cg, seed=3) <= TOL


def test_beta_zero_ignores_garbage_c(cuda):
    """test_core.cpp:264-275: beta == 0 must not read C (NaN garbage stays out)."""
    import torch
    from paper_1604_01416_b200 import local_gemm
    A = torch.rand(64, 48, device=cuda)
    B = torch.rand(48, 80, device=cuda)
    C = torch.full((64, 80), float("nan"), device=cuda)
    local_gemm(1.0, A, False, B, False, 0.0, C)
    torch.cuda.synchronize()
    assert torch.isfinite(C).all()
    assert _relfro(C, A.double() @ B.double()) <= TOL


def test_k_zero_scales_c(cuda):
    import torch
    from paper_1604_01416_b200 import local_gemm
    A = torch.empty(16, 0, device=cuda)
    B = torch.empty(0, 8, device=cuda)
    C = torch.ones(16, 8, device=cuda)
    local_gemm(2.0, A, False, B, False, 0.5, C)
    torch.cuda.synchronize()
    assert torch.equal(C, torch.full_like(C, 0.5))


@pytest.mark.parametrize("cg", [1, 2])
@pytest.mark.parametrize("k", [16384, 32768])
def test_large_k_accuracy(cuda, mode, cg, k):
    """fp32-level accuracy at the BASELINE K (1xTF32 sits near 2.5e-4; a single
    truncating TMEM accumulator near 1e-4).  The reference's own fp32
    k-ascending loop is ~3e-6 from exact at K=32768."""
    assert _run(cuda, 512, 512, k, False, False, 1.0, 0.0, cg, seed=7) <= 3e-6


@pytest.mark.parametrize("trans", [0, 1, 2, 3])
@pytest.mark.parametrize("m,n,k", [(128, 128, 8192), (4096, 64, 9216), (200, 72, 3000), (64, 1024, 4096)])
def test_split_k_shapes(cuda, mode, trans, m, n, k):
    # few output tiles, long K: split-K work items, partials summed in fixed order
    ta, tb = bool(trans & 1), bool(trans & 2)
    assert _run(cuda, m, n, k, ta, tb, 1.5, -0.5, 0, seed=trans) <= TOL


def test_split_k_deterministic(cuda):
    import torch
    from paper_1604_01416_b200 import local_gemm
    g = torch.Generator(device="cpu").manual_seed(3)
    A = (torch.rand((256, 8192), generator=g) * 2 - 1).to(cuda)
    B = (torch.rand((8192, 96), generator=g) * 2 - 1).to(cuda)
    outs = []
    for _ in range(3):
        C = torch.zeros((256, 96), device=cuda)
        local_gemm(1.0, A, False, B, False, 0.0, C)
        outs.append(C.cpu())
    assert all(torch.equal(outs[0], o) for o in outs[1:])


@pytest.mark.parametrize("gemm_mode", ["mixed", "3xtf32", "f16x2"])
def test_explicit_gemm_mode(cuda, gemm_mode):
    """The split-product scheme chosen through the ABI (dm_gemm_mode), not the
    environment: both schemes meet the fp32 bar."""
    import torch
    from paper_1604_01416_b200 import local_gemm
    g = torch.Generator(device="cpu").manual_seed(11)
    A = (torch.rand((700, 1300), generator=g) * 2 - 1).to(cuda)
    B = (torch.rand((1300, 900), generator=g) * 2 - 1).to(cuda)
    C = torch.zeros((700, 900), device=cuda)
    local_gemm(1.0, A, False, B, False, 0.0, C, gemm_mode=gemm_mode)
    torch.cuda.synchronize()
    assert _relfro(C, A.double() @ B.double()) <= 3e-6


def test_stream_ordered_on_two_streams(cuda):
    """dm_local_gemm_f32 only enqueues (no host wait, kernels.hpp:81-89 as a
    stream-ordered seam): the call returns before its GEMM ran, and two calls
    on two streams both land correctly while sharing the scratch pool."""
    import torch
    from paper_1604_01416_b200 import local_gemm
    g = torch.Generator(device="cpu").manual_seed(5)
    n = 8192
    A = [(torch.rand((n, n), generator=g) * 2 - 1).to(cuda) for _ in range(2)]
    B = (torch.rand((n, n), generator=g) * 2 - 1).to(cuda)
    C = [torch.zeros((n, n), device=cuda) for _ in range(2)]
    streams = [torch.cuda.Stream() for _ in range(2)]
    local_gemm(1.0, A[0], False, B, False, 0.0, C[0])  # warm-up (pool, attributes)
    torch.cuda.synchronize()
    done = []
    for i in range(2):
        local_gemm(1.0, A[i], False, B, False, 0.0, C[i], stream=streams[i].cuda_stream)
        ev = torch.cuda.Event()
        ev.record(streams[i])
        done.append(ev)
    # ~3 ms of tensor-core work per call: still running when the calls returned
    assert not done[1].query()
    torch.cuda.synchronize()
    Bd = B.double()
    for i in range(2):
        rows = torch.arange(0, n, 509, device=cuda)
        want = A[i][rows].double() @ Bd
        assert _relfro(C[i][rows], want) <= 3e-6


def test_cuda_graph_capture_with_workspace(cuda):
    """dm_local_gemm_f32_ws: caller-owned scratch, so the seam is capturable in
    a CUDA graph and each replay recomputes from the operands' current
    contents; the pool-backed entry refuses capture loudly."""
    import torch
    from paper_1604_01416_b200 import UsageError, local_gemm, local_gemm_workspace_size
    g = torch.Generator(device="cpu").manual_seed(8)
    m, n, k = 1024, 768, 2048
    A = (torch.rand((k, m), generator=g) * 2 - 1).to(cuda)  # op(A) = A^T
    B = (torch.rand((k, n), generator=g) * 2 - 1).to(cuda)
    C0 = (torch.rand((m, n), generator=g) * 2 - 1).to(cuda)
    C = C0.clone()
    ws = torch.empty(local_gemm_workspace_size(m, n, k), dtype=torch.uint8, device=cuda)
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):  # warm-up outside the capture
        local_gemm(1.5, A, True, B, False, -0.5, C, stream=st.cuda_stream, workspace=ws)
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        cs = torch.cuda.current_stream().cuda_stream
        local_gemm(1.5, A, True, B, False, -0.5, C, stream=cs, workspace=ws)
        with pytest.raises(UsageError):
            local_gemm(1.5, A, True, B, False, -0.5, C, stream=cs)
    for scale in (1.0, -2.0):
        A.mul_(scale)
        C.copy_(C0)
        graph.replay()
        torch.cuda.synchronize()
        want = 1.5 * (A.double().T @ B.double()) - 0.5 * C0.double()
        assert _relfro(C, want) <= 3e-6


@pytest.mark.parametrize("shape", [(4096, 1024, 2048), (1000, 744, 1304), (384, 520, 4104), (77, 96, 1004),
                                   (130, 33, 260)])
def test_f16x2_split_kernels_agree(cuda, monkeypatch, shape):
    """The f16x2 transposing split (split_trans_f16x2_kernel, swizzled smem
    tile, 16-B plane stores) writes the same planes as the tf32-shaped
    transposing kernel: a GEMM whose op(B) needs the transpose (B not
    transposed) and whose op(A) too (A transposed) is bit-identical either way."""
    import numpy as np
    import torch
    from paper_1604_01416_b200 import local_gemm
    m, n, k = shape
    g = torch.Generator(device="cuda").manual_seed(m + n + k)
    A = torch.rand(k, m, device="cuda", generator=g) * 2 - 1   # op(A) = A^T: transposing split
    B = torch.rand(k, n, device="cuda", generator=g) * 2 - 1   # op(B)^T rows = columns of B
    # ... and the direct splits: op(A) = A2 (rows), op(B) = B2^T (rows of B2)
    A2 = torch.rand(m, k, device="cuda", generator=g) * 2 - 1
    B2 = torch.rand(n, k, device="cuda", generator=g) * 2 - 1
    out = {}
    for t16 in ("1", "0"):
        monkeypatch.setenv("DM_SPLIT_TRANS16", t16)
        monkeypatch.setenv("DM_SPLIT_DIRECT16", t16)
        C = torch.zeros(m, n, device="cuda")
        local_gemm(1.0, A, True, B, False, 0.0, C, gemm_mode="f16x2")
        C2 = torch.zeros(m, n, device="cuda")
        local_gemm(1.0, A2, False, B2, True, 0.0, C2, gemm_mode="f16x2")
        torch.cuda.synchronize()
        out[t16] = C.cpu().numpy()
        out["d" + t16] = C2.cpu().numpy()
    assert out["1"].tobytes() == out["0"].tobytes()
    assert out["d1"].tobytes() == out["d0"].tobytes()
    ref = A.double().T.cpu().numpy() @ B.double().cpu().numpy()
    assert np.linalg.norm(out["1"] - ref) / np.linalg.norm(ref) <= 1e-5
