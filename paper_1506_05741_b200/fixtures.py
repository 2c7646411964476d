"""Synthetic-target fixtures at benchmark sizes (DIAMTGT v1 files).

The reference builds targets with a cyclic-Jacobi eigensolver
(proj/src/linalg.cpp:178-250), which needs minutes at d=1024 and hours at
d>=2048. For the benchmark configurations both implementations
instead load the same DIAMTGT file written here: the precision is
P = A A^T + I (pi1) or A A^T / d + I (pi2) with A drawn from the same Philox
stream (seed, 0, "target") the reference uses (proj/src/target.cpp:18-31),
the covariance is P^{-1}, and the eigenpairs come from LAPACK (numpy.eigh),
ascending, with the reference's sign convention (largest-|component|
positive, proj/src/linalg.cpp:238-247). Twisted kinds (pi5/pi6) follow
proj/src/target.cpp:112-150 on top of that base.
"""
from __future__ import annotations

import struct

import numpy as np

M0, M1 = np.uint64(0xD2511F53), np.uint64(0xCD9E8D57)
W0, W1 = np.uint64(0x9E3779B9), np.uint64(0xBB67AE85)
MASK = np.uint64(0xFFFFFFFF)


def _splitmix(state: int):
    state = (state + 0x9E3779B97F4A7C15) & (2**64 - 1)
    z = state
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & (2**64 - 1)
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & (2**64 - 1)
    return state, z ^ (z >> 31)


def _fnv1a(s: str) -> int:
    h = 0xcbf29ce484222325
    for ch in s.encode():
        h = ((h ^ ch) * 0x100000001b3) & (2**64 - 1)
    return h


def philox_key(seed: int, idx: int, purpose: str):
    s, k = _splitmix(seed)
    s, z = _splitmix(s)
    ident = z ^ ((idx * 0xA24BAED4963EE407) & (2**64 - 1)) ^ _fnv1a(purpose)
    _, sid = _splitmix(ident)
    return k & 0xFFFFFFFF, k >> 32, sid & 0xFFFFFFFF, sid >> 32


def philox_normals(seed: int, idx: int, purpose: str, start: int, n: int) -> np.ndarray:
    """n standard normals of stream (seed, idx, purpose) from draw `start` (rng.cpp:85-94)."""
    k0, k1, s0, s1 = (np.uint64(v) for v in philox_key(seed, idx, purpose))
    ctr = np.arange(start, start + n, dtype=np.uint64)
    c0 = ctr & MASK
    c1 = ctr >> np.uint64(32)
    c2 = np.full(n, s0, dtype=np.uint64)
    c3 = np.full(n, s1, dtype=np.uint64)
    for _ in range(10):
        p0 = M0 * c0
        p1 = M1 * c2
        n0 = (p1 >> np.uint64(32)) ^ c1 ^ k0
        n2 = (p0 >> np.uint64(32)) ^ c3 ^ k1
        c0, c1, c2, c3 = n0 & MASK, p1 & MASK, n2 & MASK, p0 & MASK
        k0 = (k0 + W0) & MASK
        k1 = (k1 + W1) & MASK
    w0 = (c1 << np.uint64(32)) | c0
    w1 = (c3 << np.uint64(32)) | c2
    u1 = ((w0 >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0**-53
    u2 = (w1 >> np.uint64(11)).astype(np.float64) * 2.0**-53
    return np.sqrt(-2.0 * np.log(u1)) * np.cos(6.283185307179586476925286766559 * u2)


def _sign_fix(vecs: np.ndarray) -> np.ndarray:
    idx = np.argmax(np.abs(vecs), axis=0)
    sgn = np.where(vecs[idx, np.arange(vecs.shape[1])] < 0, -1.0, 1.0)
    return vecs * sgn


KINDS = {"pi1": 0, "pi2": 1, "pi3": 2, "pi4": 3, "pi5": 4, "pi6": 5}


def build(kind: str, d: int, seed: int, twist_b: float = -1.0):
    rank = d // 10 if kind == "pi3" else d
    a = philox_normals(seed, 0, "target", 0, d * rank).reshape(d, rank)
    prec = a @ a.T
    if kind == "pi2":
        prec /= d
    prec[np.diag_indices(d)] += 1.0
    cov = np.linalg.inv(prec)
    cov = 0.5 * (cov + cov.T)
    vals, vecs = np.linalg.eigh(cov)
    vecs = _sign_fix(vecs)
    out = dict(kind=KINDS[kind], dim=d, seed=seed, sigma2=0.0, twist_b=0.0, precision=prec, covariance=cov,
               eigvecs=vecs, eigvals=vals, b_coeffs=np.zeros(d), mean=np.zeros(d), eigen_mean=np.zeros(d),
               eigen_var=vals.copy())
    if kind in ("pi5", "pi6"):
        assert d % 20 == 0, "twisted targets need d divisible by 20"
        b = twist_b if twist_b >= 0 else (0.3 if kind == "pi5" else 2.0)
        m = d // 10
        bc = np.zeros(d)
        for i in range(1, m, 2):
            bc[i - 1] = b / (vals[i - 1] * np.sqrt(d))
        em, ev = np.zeros(d), vals.copy()
        for i in range(2, m + 1, 2):
            em[i - 1] = -bc[i - 2] * vals[i - 2]
            ev[i - 1] = vals[i - 1] + 2.0 * bc[i - 2] ** 2 * vals[i - 2] ** 2
        out.update(kind=KINDS[kind], twist_b=b, precision=np.zeros((0, 0)), b_coeffs=bc, eigen_mean=em,
                   eigen_var=ev, mean=vecs @ em, covariance=(vecs * ev) @ vecs.T)
    elif kind not in ("pi1", "pi2", "pi3"):
        raise ValueError(f"fixture kind {kind} not supported")
    return out


def write(path: str, t: dict) -> None:
    def mat(x):
        x = np.ascontiguousarray(x, dtype="<f8")
        r, c = x.shape
        return struct.pack("<QQ", r, c) + x.tobytes()

    def vec(x):
        x = np.ascontiguousarray(x, dtype="<f8")
        return struct.pack("<Q", x.size) + x.tobytes()

    blob = b"DIAMTGT\0" + struct.pack("<III", 1, 0x01020304, t["kind"]) + struct.pack("<QQ", t["dim"], t["seed"])
    blob += struct.pack("<dd", t["sigma2"], t["twist_b"])
    blob += mat(t["precision"]) + mat(t["covariance"]) + mat(t["eigvecs"])
    for key in ("eigvals", "b_coeffs", "mean", "eigen_mean", "eigen_var"):
        blob += vec(t[key])
    with open(path, "wb") as f:
        f.write(blob)


def make(path: str, kind: str, d: int, seed: int, twist_b: float = -1.0) -> str:
    write(path, build(kind, d, seed, twist_b))
    return path
