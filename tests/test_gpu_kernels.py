"""Unit checks of the build-time dense kernels (csrc/dgemm.inc,
csrc/dense_inv.inc) through the C ABI against torch fp64 references.  These
are the contractions behind the exact local solves (reading R6; T_ML,
P:861): the DMMA GEMM must agree with a plain fp64 GEMM to rounding, and the
pivoted Gauss-Jordan inverse must invert matrices that need pivoting."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,k,batch", [(64, 64, 16, 1), (1, 1, 1, 3), (70, 33, 129, 2), (257, 130, 64, 1),
                                         (5, 300, 7, 4), (1024, 512, 256, 1),
                                         (300, 200, 77, 2), (192, 130, 50, 3), (130, 129, 51, 2),
                                         (96, 96, 2, 1), (128, 256, 18, 2)])
@pytest.mark.parametrize("transA", [False, True])
@pytest.mark.parametrize("beta", [0.0, 1.0, -0.5])
def test_dgemm_matches_torch(m, n, k, batch, transA, beta):
    from paper_2510_22077_b200._lib import dgemm
    g = torch.Generator(device="cuda").manual_seed(m * 7 + n * 3 + k)
    A = torch.randn((batch, m, k) if transA else (batch, k, m), dtype=torch.float64, device="cuda", generator=g)
    B = torch.randn((batch, n, k), dtype=torch.float64, device="cuda", generator=g)
    C = torch.randn((batch, n, m), dtype=torch.float64, device="cuda", generator=g)
    opA_t = A.transpose(1, 2) if transA else A          # (batch, k, m) = op(A)^T
    ref = -1.25 * torch.bmm(B, opA_t) + beta * C          # C^T = B^T op(A)^T
    dgemm(A, B, C, alpha=-1.25, beta=beta, transA=transA)
    torch.cuda.synchronize()
    err = (C - ref).abs().max().item()
    scale = (torch.bmm(B.abs(), opA_t.abs())).max().item()
    assert err <= 1e-14 * k * max(scale, 1.0)


@pytest.mark.parametrize("n", [1, 2, 31, 32, 33, 100, 257])
def test_dense_inverse_pivoted(n):
    """A matrix whose leading entries are zero (no unpivoted elimination
    exists) and a permutation-scrambled diagonally dominant one."""
    from paper_2510_22077_b200._lib import dense_inverse
    rng = np.random.default_rng(n)
    M = rng.standard_normal((n, n)) + n * np.eye(n)
    perm = rng.permutation(n)
    M = M[perm]                                         # zero-free diagonal not guaranteed
    if n > 1:
        M[0, 0] = 0.0
    A = torch.tensor(M, dtype=torch.float64, device="cuda")
    dense_inverse(A)
    X = A.cpu().numpy()
    I = np.eye(n)
    assert np.abs(M @ X - I).max() <= 1e-10
    S = np.zeros((3, 3))
    with pytest.raises(Exception):
        dense_inverse(torch.tensor(S, dtype=torch.float64, device="cuda"))
