"""Kernel-level parity on the B200, through the C ABI (include/diam_b200.h).

Each sm_100a kernel is checked against the CPU oracle (oracle/diam_oracle.c)
or an exact reference on the same inputs:
  * Philox draws: raw u64 and uniform_open BIT-EXACT (integer arithmetic);
    normals within a stated ulp bound (CUDA libm vs glibc log/cos);
  * FP64 DMMA GEMM (all layouts, triangular modes, ragged sizes):
    rel. Frobenius error <= 1e-13 vs a float64 reference;
  * batched POTRF: vs the oracle's cholesky, ||L - L_ref||_F/||L_ref||_F <=
    1e-10 * max(1, cond/1e3) and reconstruction <= 1e-10,
    not-positive-definite detection;
  * batched TRSV: vs the oracle's tri_solve, rel. error <= 1e-12 * cond-scale.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
GOLD = os.path.join(os.path.dirname(__file__), "golden")


def ptr(t):
    return C.c_void_p(t.data_ptr())


def cu(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture(scope="module")
def lib(b200):
    assert torch.cuda.is_available()
    return b200


# ------------------------------------------------------------------ draws
def test_draws_u64_and_uniform_bit_exact(lib):
    n = 1 << 16
    out = torch.zeros(n, dtype=torch.int64, device="cuda")
    lib.check(lib.lib.diamx_draws(0, None, ptr(out), n, 42, 0, b"noise", 0, None))
    got = out.cpu().numpy().view(np.uint64)
    g = json.load(open(os.path.join(GOLD, "rng.json")))
    assert [int(v) for v in got[:4]] == [int(v) for v in g["u64_test_rng_cpp"]]
    assert np.array_equal(got, O.fill("u64", 42, 0, "noise", 0, n))
    u = torch.zeros(n, dtype=torch.float64, device="cuda")
    lib.check(lib.lib.diamx_draws(1, ptr(u), None, n, 7, 3, b"uniform", 100, None))
    assert np.array_equal(u.cpu().numpy(), O.fill("uniform_open", 7, 3, "uniform", 100, n))


def test_normals_ulp_bound(lib):
    n = 1 << 18
    z = torch.zeros(n, dtype=torch.float64, device="cuda")
    lib.check(lib.lib.diamx_draws(2, ptr(z), None, n, 9, 3, b"noise", 17, None))
    got = z.cpu().numpy()
    ref = O.fill("normal", 9, 3, "noise", 17, n)
    ulp = np.abs(got.view(np.int64) - ref.view(np.int64))
    frac_exact = float(np.mean(ulp == 0))
    print(f"normals: {frac_exact:.4f} bit-exact, max ulp {ulp.max()}, p99.9 {np.quantile(ulp, 0.999)}")
    # |Δ| relative to the value: log (1 ulp) and cos (2 ulp) errors of CUDA's libm,
    # amplified only where cos(2πu) is near zero
    rel = np.abs(got - ref) / np.maximum(np.abs(ref), 1e-300)
    assert np.quantile(rel, 0.999) < 1e-14
    assert np.max(np.abs(got - ref)) < 1e-13
    assert abs(got.mean()) < 0.01 and abs(got.var() - 1) < 0.01


# ------------------------------------------------------------------ GEMM
def run_gemm(lib, A, B, Cm, m, n, k, ak, bk, alpha, beta, trib=0, tric=0):
    lda = A.shape[1]
    ldb = B.shape[1]
    ldc = Cm.shape[1]
    lib.check(lib.lib.diamx_gemm(ptr(A), ptr(B), ptr(Cm), m, n, k, lda, ldb, ldc, int(ak), int(bk), alpha, beta,
                                 trib, tric, None))


@pytest.mark.parametrize("ak", [True, False])
@pytest.mark.parametrize("bk", [True, False])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (77, 50, 33), (300, 260, 129), (8, 1030, 517)])
def test_gemm_layouts(lib, ak, bk, m, n, k):
    rng = np.random.default_rng(m + n + k)
    pad = lambda x: (x + 7) // 8 * 8  # noqa: E731
    a = rng.normal(size=(m, k))
    b = rng.normal(size=(k, n))
    c0 = rng.normal(size=(m, n))
    A = np.zeros((m, pad(k))) if ak else np.zeros((k, pad(m)))
    if ak:
        A[:, :k] = a
    else:
        A[:, :m] = a.T
    B = np.zeros((n, pad(k))) if bk else np.zeros((k, pad(n)))
    if bk:
        B[:, :k] = b.T
    else:
        B[:, :n] = b
    Cm = np.zeros((m, pad(n)))
    Cm[:, :n] = c0
    Ad, Bd, Cd = cu(A), cu(B), cu(Cm)
    run_gemm(lib, Ad, Bd, Cd, m, n, k, ak, bk, 0.75, -0.5)
    want = 0.75 * (a @ b) - 0.5 * c0
    got = Cd.cpu().numpy()
    assert np.linalg.norm(got[:, :n] - want) / np.linalg.norm(want) < 1e-13
    assert np.all(got[:, n:] == 0)  # pad columns untouched


def test_gemm_triangular_modes(lib):
    rng = np.random.default_rng(5)
    d, rows = 200, 96
    ld = 200
    Lm = np.tril(rng.normal(size=(d, d)))
    W = rng.normal(size=(rows, d))
    Xi = cu(np.zeros((rows, ld)))
    # TRMM: Xi = W L^T with B lower-triangular (K loop clipped per n-tile)
    run_gemm(lib, cu(W), cu(Lm), Xi, rows, d, d, True, True, 1.0, 0.0, trib=1)
    want = W @ Lm.T
    assert np.linalg.norm(Xi.cpu().numpy() - want) / np.linalg.norm(want) < 1e-13
    # SYRK: S = a X^T X + b S on the lower triangle only
    X = rng.normal(size=(rows, d))
    S0 = np.tril(rng.normal(size=(d, d)))
    Sd = cu(S0.copy())
    run_gemm(lib, cu(X), cu(X), Sd, d, d, rows, False, False, 0.25, 0.5, tric=1)
    got = Sd.cpu().numpy()
    want = np.tril(0.25 * X.T @ X + 0.5 * S0)
    assert np.linalg.norm(np.tril(got) - want) / np.linalg.norm(want) < 1e-13
    assert np.array_equal(np.triu(got, 1), np.triu(S0, 1))  # upper part never written


# ------------------------------------------------------------------ POTRF
def oracle_chol(m):
    L = O.oracle()
    L.or_cholesky.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p]
    m = np.ascontiguousarray(m)
    out = np.zeros_like(m)
    st = L.or_cholesky(m.ctypes.data, m.shape[0], out.ctypes.data)
    return st, out


@pytest.mark.parametrize("d", [1, 5, 63, 64, 65, 127, 128, 129, 130, 191, 192, 193, 257, 520, 1024])
def test_potrf_batched_vs_oracle(lib, d):
    # the blocked POTRF at every block-column shape: one or two 64-wide diagonal blocks per
    # 128-wide block column, ragged and narrow last block columns
    rng = np.random.default_rng(d)
    batch = 3
    ld = (d + 7) // 8 * 8
    mats, host = [], np.zeros((batch, d, ld))
    for i in range(batch):
        a = rng.normal(size=(d, d + 3))
        m = a @ a.T / d + (0.1 + i) * np.eye(d)
        mats.append(m)
        host[i, :, :d] = np.tril(m)
    A = cu(host)
    status = torch.zeros(batch, dtype=torch.int32, device="cuda")
    lib.check(lib.lib.diamx_potrf(ptr(A), d * ld, ld, d, batch, ptr(status), None))
    assert status.cpu().numpy().tolist() == [0] * batch
    got = A.cpu().numpy()
    for i, m in enumerate(mats):
        st, lref = oracle_chol(m)
        assert st == 0
        lg = got[i, :, :d]
        assert np.array_equal(np.triu(lg, 1), np.zeros((d, d)))
        cond = np.linalg.cond(m)
        assert np.linalg.norm(lg - lref) / np.linalg.norm(lref) <= 1e-10 * max(1.0, cond / 1e3)
        assert np.linalg.norm(lg @ lg.T - m) / np.linalg.norm(m) <= 1e-10


@pytest.mark.parametrize("d", [1024, 1089])
def test_potrf_default_path_large(lib, d):
    # the default (fused) factorization at the bench dimension and at a ragged size whose
    # last block column is narrow (1089 = 8 x 128 + 65)
    rng = np.random.default_rng(d)
    batch = 2
    ld = (d + 7) // 8 * 8
    mats, host = [], np.zeros((batch, d, ld))
    for i in range(batch):
        a = rng.normal(size=(d, d + 16))
        m = a @ a.T / d + (0.5 + i) * np.eye(d)
        mats.append(m)
        host[i, :, :d] = np.tril(m)
    A = cu(host)
    status = torch.zeros(batch, dtype=torch.int32, device="cuda")
    lib.check(lib.lib.diamx_potrf(ptr(A), d * ld, ld, d, batch, ptr(status), None))
    assert status.cpu().numpy().tolist() == [0] * batch
    got = A.cpu().numpy()
    for i, m in enumerate(mats):
        st, lref = oracle_chol(m)
        assert st == 0
        lg = got[i, :, :d]
        assert np.array_equal(np.triu(lg, 1), np.zeros((d, d)))
        assert np.linalg.norm(lg - lref) / np.linalg.norm(lref) <= 1e-12
        assert np.linalg.norm(lg @ lg.T - m) / np.linalg.norm(m) <= 1e-12


def test_potrf_detects_not_positive_definite(lib):
    d, ld = 100, 104
    rng = np.random.default_rng(1)
    q, _ = np.linalg.qr(rng.normal(size=(d, d)))
    ev = np.linspace(1, 2, d)
    ev[70] = -0.5
    bad = (q * ev) @ q.T
    good = q @ np.diag(np.linspace(1, 2, d)) @ q.T
    host = np.zeros((2, d, ld))
    host[0, :, :d] = np.tril(bad)
    host[1, :, :d] = np.tril(good)
    A = cu(host)
    status = torch.zeros(2, dtype=torch.int32, device="cuda")
    lib.check(lib.lib.diamx_potrf(ptr(A), d * ld, ld, d, 2, ptr(status), None))
    assert status.cpu().numpy().tolist() == [1, 0]
    assert oracle_chol(bad)[0] == 4


# ------------------------------------------------------------------ TRSV
@pytest.mark.parametrize("d", [3, 64, 100, 1000])
def test_trsv_vs_oracle(lib, d):
    rng = np.random.default_rng(d)
    ld = (d + 7) // 8 * 8
    batch = 2
    Lh = np.zeros((batch, d, ld))
    xs = np.zeros((batch, ld))
    for i in range(batch):
        a = rng.normal(size=(d, d + 2))
        _, l = oracle_chol(a @ a.T / d + np.eye(d))
        Lh[i, :, :d] = l
        xs[i, :d] = rng.normal(size=d)
    Ld, Xd = cu(Lh), cu(xs)
    Yd = torch.zeros_like(Xd)
    Q = torch.zeros(batch, dtype=torch.float64, device="cuda")
    lib.check(lib.lib.diamx_trsv(ptr(Ld), d * ld, ld, ptr(Xd), ptr(Yd), ptr(Q), d, batch, None))
    L = O.oracle()
    L.or_tri_solve.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    y = Yd.cpu().numpy()
    q = Q.cpu().numpy()
    for i in range(batch):
        l = np.ascontiguousarray(Lh[i, :, :d])
        x = np.ascontiguousarray(xs[i, :d])
        yr = np.zeros(d)
        assert L.or_tri_solve(l.ctypes.data, d, x.ctypes.data, yr.ctypes.data) == 0
        assert np.linalg.norm(y[i, :d] - yr) / np.linalg.norm(yr) < 1e-12
        assert abs(q[i] - 0.5 * yr @ yr) / (0.5 * yr @ yr) < 1e-12


# ------------------------------------------------------------------ target builder (large d)
@pytest.mark.parametrize("kind", ["pi1", "pi2", "pi3", "pi4", "pi5", "pi6"])
def test_gpu_target_builder_matches_host(b200, tmp_path, monkeypatch, kind):
    """diam_target_build's GPU path (DMMA Gram/products + cuSOLVER eigensolver) against the
    host restatement, which is bit-identical to the reference's builder."""
    d, seed = 200, 3
    h = b200.target_build(kind, d, seed)  # d < 1024: host path
    ph = str(tmp_path / "h.bin")
    h.save(ph)
    monkeypatch.setenv("DIAM_B200_TARGET_BUILD", "gpu")
    g = b200.target_build(kind, d, seed)
    pg = str(tmp_path / "g.bin")
    g.save(pg)
    a, b = O.read_target(ph), O.read_target(pg)
    assert (a.kind, a.dim, a.seed) == (b.kind, b.dim, b.seed)
    rel = lambda x, y: np.linalg.norm(x - y) / max(np.linalg.norm(y), 1e-300)
    if a.precision.size:
        assert rel(b.precision, a.precision) <= (1e-12 if kind in ("pi1", "pi2", "pi3") else 1e-10)
    assert rel(b.covariance, a.covariance) <= 1e-10
    assert np.max(np.abs(b.eigvals - a.eigvals) / a.eigvals) <= 1e-10
    # eigenvectors: same sign convention, accuracy ~ eps / relative gap; inside a
    # repeated eigenvalue (pi3: rank d/10 + I) only the invariant subspace is defined
    lam = a.eigvals
    start = 0
    while start < d:
        end = start + 1
        while end < d and lam[end] - lam[end - 1] <= 1e-9 * lam[end]:
            end += 1
        va, vb = a.eigvecs[:, start:end], b.eigvecs[:, start:end]
        if end - start == 1:
            assert np.max(np.abs(vb - va)) <= 1e-8
        else:
            assert np.max(np.abs(vb @ vb.T - va @ va.T)) <= 1e-8
        start = end
    assert np.max(np.abs(b.mean - a.mean)) <= 1e-10 * max(1.0, np.max(np.abs(a.mean)))
    assert rel(b.eigen_var, a.eigen_var) <= 1e-10
    assert np.array_equal(b.b_coeffs == 0, a.b_coeffs == 0)


def test_gpu_target_builder_large_d(b200, tmp_path):
    """d >= 1024 goes to the GPU builder by default: a d=2048 pi1 target in seconds
    (the reference's Jacobi takes hours), internally consistent."""
    import time
    t0 = time.perf_counter()
    t = b200.target_build("pi1", 2048, 7)
    secs = time.perf_counter() - t0
    p = str(tmp_path / "t.bin")
    t.save(p)
    td = O.read_target(p)
    P, Cv, V, lam = td.precision, td.covariance, td.eigvecs, td.eigvals
    print(f"d=2048 target build {secs:.1f} s")
    assert secs < 120
    assert np.all(np.diff(lam) >= 0) and lam[0] > 0
    assert np.linalg.norm(P @ Cv - np.eye(2048)) <= 1e-9 * np.sqrt(2048)
    assert np.linalg.norm(V.T @ V - np.eye(2048)) <= 1e-10 * 2048
    assert np.linalg.norm(Cv @ V - V * lam) <= 1e-10 * np.linalg.norm(Cv)
    idx = np.argmax(np.abs(V), axis=0)
    assert np.all(V[idx, np.arange(2048)] > 0)
