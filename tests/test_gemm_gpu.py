"""K-GEMM parity: complex128 DMMA GEMM vs NumPy (zgemm), all op combinations,
ragged shapes, batching, permuted stores and split-K.  Floating point:
tolerance 1e-13 relative Frobenius."""
import numpy as np
import pytest

from paper_2212_09782_b200.qrtebd import zgemm

pytestmark = pytest.mark.gpu


def crand(rng, *shape):
    return rng.standard_normal(shape) + 1j * rng.standard_normal(shape)


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def op(x, o):
    return x if o == 0 else x.conj().T


@pytest.mark.parametrize("opa,opb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(64, 128, 16), (37, 53, 29), (5, 7, 3), (200, 130, 300), (1, 1, 1),
                                   (32, 300, 1000), (25, 64, 25),
                                   # makespan-model shapes: split-K over 64 x 128 tiles, K = 32 updates
                                   (1280, 256, 1280), (2000, 300, 32)])
def test_zgemm_ops(ctx, opa, opb, m, n, k):
    rng = np.random.default_rng(m * 1000 + n * 10 + k + 7 * opa + 13 * opb)
    a = crand(rng, *((m, k) if opa == 0 else (k, m)))
    b = crand(rng, *((k, n) if opb == 0 else (n, k)))
    c0 = crand(rng, m, n)
    ta, tb, tc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(c0)
    zgemm(ctx, opa, opb, m, n, k, ta.ptr, a.shape[1], tb.ptr, b.shape[1], tc.ptr, n, alpha=-0.5, beta=2.0)
    ref = -0.5 * op(a, opa) @ op(b, opb) + 2.0 * c0
    assert rel(tc.numpy(), ref) < 1e-13


def test_zgemm_batched_shared_a(ctx):
    rng = np.random.default_rng(3)
    m, n, k, nb = 50, 70, 40, 5
    a = crand(rng, m, k)
    b = crand(rng, nb, k, n)
    ta, tb, tc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(np.zeros((nb, m, n)))
    zgemm(ctx, 0, 0, m, n, k, ta.ptr, k, tb.ptr, n, tc.ptr, n, batch=nb, stride_a=0, stride_b=k * n,
          stride_c=m * n)
    ref = np.einsum("mk,bkn->bmn", a, b)
    assert rel(tc.numpy(), ref) < 1e-13


def test_zgemm_split_k_deterministic(ctx):
    # tall-K skinny output triggers split-K; result must be bitwise reproducible
    rng = np.random.default_rng(11)
    m, n, k = 32, 96, 6000
    a = crand(rng, k, m)
    b = crand(rng, k, n)
    ta, tb = ctx.tensor(a), ctx.tensor(b)
    outs = []
    for _ in range(2):
        tc = ctx.tensor(np.zeros((m, n)))
        zgemm(ctx, 1, 0, m, n, k, ta.ptr, m, tb.ptr, n, tc.ptr, n)
        outs.append(tc.numpy())
    assert rel(outs[0], a.conj().T @ b) < 1e-13
    assert np.array_equal(outs[0], outs[1])


@pytest.mark.parametrize("opa,opb", [(0, 0), (0, 1), (1, 0), (1, 1)])
def test_zgemm_3m_unbalanced_parts(ctx, opa, opb):
    """The 3M products (Im c = P3 - P1 - P2) keep the normwise bound
    |dC| <= c u |A||B| K even when real and imaginary parts differ by orders
    of magnitude, and real inputs give exactly real outputs."""
    rng = np.random.default_rng(31 + 2 * opa + opb)
    m, n, k = 300, 260, 700
    a = rng.standard_normal((m, k)) + 1j * 1e-4 * rng.standard_normal((m, k))
    b = 1e-3 * rng.standard_normal((k, n)) + 1j * rng.standard_normal((k, n))
    ast, bst = op(a, opa), op(b, opb)  # stored so that op(stored) = a, b
    ta, tb, tc = ctx.tensor(ast.copy()), ctx.tensor(bst.copy()), ctx.tensor(np.zeros((m, n)) + 0j)
    zgemm(ctx, opa, opb, m, n, k, ta.ptr, ast.shape[1], tb.ptr, bst.shape[1], tc.ptr, n, alpha=1.0, beta=0.0)
    ref = a @ b
    bound = np.abs(a).max() * np.abs(b).max() * k * 2.2e-16
    assert np.abs(tc.numpy() - ref).max() < 4 * bound
    # real operands: the imaginary parts cancel exactly (P3 and P1 see the same inputs)
    ar, br = rng.standard_normal((m, k)) + 0j, rng.standard_normal((k, n)) + 0j
    ta, tb = ctx.tensor(op(ar, opa).copy()), ctx.tensor(op(br, opb).copy())
    zgemm(ctx, opa, opb, m, n, k, ta.ptr, m if opa else k, tb.ptr, k if opb else n, tc.ptr, n, alpha=1.0, beta=0.0)
    out = tc.numpy()
    assert np.all(out.imag == 0.0)
    assert rel(out, ar @ br) < 1e-14


@pytest.mark.parametrize("opa,opb", [(0, 0), (0, 1), (1, 0), (1, 1)])
@pytest.mark.parametrize("m,n,k", [(64, 256, 1024), (200, 136, 88), (1280, 1280, 32), (520, 96, 5120),
                                   (72, 24, 40)])
def test_zgemm_chunked_maps_batched(ctx, opa, opb, m, n, k):
    """4-D chunked tensor maps (contiguous extents multiple of 8), batched with
    both operands strided, leading dimensions wider than the matrices, and the
    two-CTA short-K tiles / split-K up to eight waves the dispatcher picks."""
    rng = np.random.default_rng(7 * m + n + 3 * k + opa + 2 * opb)
    nb = 3
    pad = 8  # ld = extent + 8: rows do not abut
    ra, ca = (m, k) if opa == 0 else (k, m)
    rb, cb = (k, n) if opb == 0 else (n, k)
    a = crand(rng, nb, ra, ca + pad)
    b = crand(rng, nb, rb, cb + pad)
    c0 = crand(rng, nb, m, n)
    ta, tb, tc = ctx.tensor(a), ctx.tensor(b), ctx.tensor(c0)
    zgemm(ctx, opa, opb, m, n, k, ta.ptr, ca + pad, tb.ptr, cb + pad, tc.ptr, n, alpha=0.5, beta=-1.0, batch=nb,
          stride_a=ra * (ca + pad), stride_b=rb * (cb + pad), stride_c=m * n)
    ref = np.stack([0.5 * op(a[i, :, :ca], opa) @ op(b[i, :, :cb], opb) - c0[i] for i in range(nb)])
    assert rel(tc.numpy(), ref) < 1e-13
