"""ctypes bindings for the CPU checker (TEST INFRASTRUCTURE).

* ``oracle/liboracle.so`` — the C restatement of the reference hot path
  (oracle/diam_oracle.c), the oracle the GPU path is checked against.
* ``oracle/_ref/libdiam_ref.so`` — the reference itself, built from
  /root/reference/proj/src by oracle/Makefile (used to pin the restatement).

Also holds a reader/writer for the reference's DIAMTGT v1 target file
(reference: proj/src/target.cpp:187-231, binio layout proj/src/binio.hpp).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this.
"""
from __future__ import annotations

import ctypes as C
import os
import struct
from dataclasses import dataclass, field

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdiam_ref.so")

_dp = C.POINTER(C.c_double)
_u64p = C.POINTER(C.c_uint64)


def dptr(a: np.ndarray):
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_dp)


# --------------------------------------------------------------------------
# structs mirrored from oracle/diam_oracle.h
# --------------------------------------------------------------------------
class OrTarget(C.Structure):
    _fields_ = [("dim", C.c_size_t), ("twisted", C.c_int), ("precision", _dp), ("eigvecs_t", _dp),
                ("eigvals", _dp), ("b_coeffs", _dp), ("proj_min", _dp), ("proj_max", _dp),
                ("covariance", _dp), ("mean", _dp)]


class OrKernelCfg(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", C.c_size_t), ("beta_init", C.c_double),
                ("inflation", C.c_double), ("adaptive_ref", C.c_int), ("n_lag", C.c_size_t),
                ("band_lo", C.c_double), ("band_hi", C.c_double), ("n0", C.c_uint64),
                ("n_ref_start", C.c_uint64), ("beta_adapt_factor", C.c_double),
                ("beta_min", C.c_double), ("beta_max", C.c_double), ("adapt_beta", C.c_int),
                ("use_explicit_inverse", C.c_int)]


class OrRunCfg(C.Structure):
    _fields_ = [("kernel", OrKernelCfg), ("chains", C.c_size_t), ("intervals_per_batch", C.c_size_t),
                ("max_batches", C.c_size_t), ("cov_tol", C.c_double), ("mean_tol", C.c_double),
                ("psrf_tol", C.c_double), ("max_samples", C.c_int64), ("init_dispersion", C.c_double),
                ("master_seed", C.c_uint64), ("record_traces", C.c_int), ("trace_thin", C.c_size_t),
                ("trace_eigen_projections", C.c_int)]


class OrRunOut(C.Structure):
    _fields_ = [("batches", C.c_size_t), ("total_samples", C.c_uint64),
                ("accumulated_samples", C.c_uint64), ("stop_reason", C.c_int),
                ("global_mean", _dp), ("global_cov", _dp), ("cov_error_hist", _dp),
                ("mean_error_hist", _dp), ("psrf_hist", _dp), ("beta_hist", _dp), ("acc_hist", _dp),
                ("accept_bits", _dp), ("log_ratio", _dp), ("log_u", _dp), ("final_x", _dp),
                ("traces", _dp), ("trace_cap", C.c_size_t), ("trace_len", C.c_size_t)]


class OrRunOpts(C.Structure):
    _fields_ = [("threads", C.c_int), ("chain_ids", C.POINTER(C.c_size_t)), ("n_ids", C.c_size_t)]


KIND = {"rw": 0, "pcn": 1, "am": 2, "diam": 3}
STOP = {0: "batch_cap", 1: "max_samples", 2: "psrf", 3: "cov_tol", 4: "mean_tol"}

_oracle = None
_ref = None


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_SO)
        lib.or_lane_dot.restype = C.c_double
        lib.or_log_density.restype = C.c_double
        lib.or_uniform_open.restype = C.c_double
        lib.or_normal.restype = C.c_double
        lib.or_next_u64.restype = C.c_uint64
        lib.or_cov_error.restype = C.c_double
        lib.or_mean_error.restype = C.c_double
        lib.or_last_error.restype = C.c_char_p
        lib.or_fill_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _u64p]
        lib.or_fill_uniform_open.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _dp]
        lib.or_fill_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _dp]
        _oracle = lib
    return _oracle


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_SO)
        lib.shim_fill_u64.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _u64p]
        lib.shim_fill_uniform_open.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _dp]
        lib.shim_fill_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_char_p, C.c_uint64, C.c_size_t, _dp]
        _ref = lib
    return _ref


# --------------------------------------------------------------------------
# draws
# --------------------------------------------------------------------------
def fill(kind: str, seed: int, idx: int, purpose: str, start: int, n: int, lib: str = "oracle"):
    """kind in {u64, uniform_open, normal}; lib in {oracle, ref}."""
    L = oracle() if lib == "oracle" else ref()
    pfx = "or_fill_" if lib == "oracle" else "shim_fill_"
    if kind == "u64":
        out = np.zeros(n, dtype=np.uint64)
        getattr(L, pfx + "u64")(seed, idx, purpose.encode(), start, n, out.ctypes.data_as(_u64p))
    else:
        out = np.zeros(n, dtype=np.float64)
        getattr(L, pfx + kind)(seed, idx, purpose.encode(), start, n, dptr(out))
    return out


# --------------------------------------------------------------------------
# DIAMTGT v1 files (proj/src/target.cpp:187-231)
# --------------------------------------------------------------------------
@dataclass
class TargetData:
    kind: int
    dim: int
    seed: int
    sigma2: float
    twist_b: float
    precision: np.ndarray
    covariance: np.ndarray
    eigvecs: np.ndarray
    eigvals: np.ndarray
    b_coeffs: np.ndarray
    mean: np.ndarray
    eigen_mean: np.ndarray
    eigen_var: np.ndarray
    _keep: list = field(default_factory=list, repr=False)

    @property
    def twisted(self) -> bool:
        return self.kind in (4, 5)

    def or_target(self) -> OrTarget:
        d = self.dim
        prec = self.precision if self.precision.size else np.zeros((d, d))
        vt = np.ascontiguousarray(self.eigvecs.T)
        pmin = np.ascontiguousarray(self.eigvecs[:, 0])
        pmax = np.ascontiguousarray(self.eigvecs[:, d - 1])
        arrs = [np.ascontiguousarray(a, dtype=np.float64) for a in
                (prec, vt, self.eigvals, self.b_coeffs, pmin, pmax, self.covariance, self.mean)]
        self._keep = arrs
        return OrTarget(d, int(self.twisted), *[dptr(a) for a in arrs])


def read_target(path: str) -> TargetData:
    with open(path, "rb") as f:
        buf = f.read()
    off = 0

    def take(fmt):
        nonlocal off
        v = struct.unpack_from("<" + fmt, buf, off)
        off += struct.calcsize("<" + fmt)
        return v[0]

    def mat():
        nonlocal off
        r, c = take("Q"), take("Q")
        a = np.frombuffer(buf, dtype="<f8", count=r * c, offset=off).reshape(r, c).copy()
        off += 8 * r * c
        return a

    def vec():
        nonlocal off
        n = take("Q")
        a = np.frombuffer(buf, dtype="<f8", count=n, offset=off).copy()
        off += 8 * n
        return a

    magic = buf[:8]
    off = 8
    assert magic == b"DIAMTGT\0", magic
    assert take("I") == 1 and take("I") == 0x01020304
    kind, dim, seed = take("I"), take("Q"), take("Q")
    sigma2, twist_b = take("d"), take("d")
    precision, covariance, eigvecs = mat(), mat(), mat()
    eigvals, b_coeffs, mean, eigen_mean, eigen_var = vec(), vec(), vec(), vec(), vec()
    return TargetData(kind, dim, seed, sigma2, twist_b, precision, covariance, eigvecs, eigvals,
                      b_coeffs, mean, eigen_mean, eigen_var)


def write_target(path: str, t: TargetData) -> None:
    def mat(a):
        a = np.ascontiguousarray(a, dtype="<f8")
        if a.ndim == 1:
            a = a.reshape(0, 0) if a.size == 0 else a
        r, c = (a.shape if a.ndim == 2 else (0, 0))
        return struct.pack("<QQ", r, c) + a.tobytes()

    def vec(a):
        a = np.ascontiguousarray(a, dtype="<f8")
        return struct.pack("<Q", a.size) + a.tobytes()

    out = b"DIAMTGT\0" + struct.pack("<III", 1, 0x01020304, t.kind) + struct.pack("<QQ", t.dim, t.seed)
    out += struct.pack("<dd", t.sigma2, t.twist_b)
    out += mat(t.precision) + mat(t.covariance) + mat(t.eigvecs)
    out += vec(t.eigvals) + vec(t.b_coeffs) + vec(t.mean) + vec(t.eigen_mean) + vec(t.eigen_var)
    with open(path, "wb") as f:
        f.write(out)


# --------------------------------------------------------------------------
# whole-run oracle (oracle/diam_oracle.c: or_run restating proj/src/runner.cpp)
# --------------------------------------------------------------------------
def kernel_cfg(kind: str, dim: int, **over) -> OrKernelCfg:
    k = OrKernelCfg()
    oracle().or_kernel_defaults(C.byref(k), KIND[kind], C.c_size_t(dim))
    for key, v in over.items():
        setattr(k, key, v)
    return k


def run(target: TargetData, kind: str = "diam", chains: int = 1, M: int = 1, K: int = 1,
        seed: int = 1, inject_w=None, record_decisions: bool = False, cov_tol=-1.0,
        mean_tol=-1.0, psrf_tol=-1.0, max_samples=-1, dispersion=1.0, threads: int = 1,
        chain_ids=None, traces: bool = False, trace_thin: int = 1, **kover):
    """or_run_ex: the whole run (proj/src/runner.cpp:216-279) on `threads` host threads.
    chain_ids: replay only those global chains (per-chain outputs of the first batch;
    inject_w then lists their windows in the same order). traces: record log pi and the
    two eigen projections (runner.cpp:363-379)."""
    d = target.dim
    cfg = OrRunCfg()
    cfg.kernel = kernel_cfg(kind, d, **kover)
    cfg.chains, cfg.intervals_per_batch, cfg.max_batches = chains, M, K
    cfg.cov_tol, cfg.mean_tol, cfg.psrf_tol, cfg.max_samples = cov_tol, mean_tol, psrf_tol, max_samples
    cfg.init_dispersion, cfg.master_seed = dispersion, seed
    cfg.record_traces, cfg.trace_thin, cfg.trace_eigen_projections = int(traces), trace_thin, int(traces)
    nl = cfg.kernel.n_lag
    nrun = len(chain_ids) if chain_ids is not None else chains
    res = dict(global_mean=np.zeros(d), global_cov=np.zeros((d, d)), cov_error_hist=np.zeros(K),
               mean_error_hist=np.zeros(K), psrf_hist=np.zeros(K), beta_hist=np.zeros((nrun, K * M)),
               acc_hist=np.zeros((nrun, K * M)), final_x=np.zeros((nrun, d)))
    if record_decisions:
        for key in ("accept_bits", "log_ratio", "log_u"):
            res[key] = np.zeros((nrun, K * M * nl))
    cap = K * M * nl
    if traces:
        res["traces"] = np.zeros((nrun, 3, cap))
    out = OrRunOut()
    for key, a in res.items():
        setattr(out, key, dptr(a))
    out.trace_cap = cap if traces else 0
    tgt = target.or_target()
    w_arr = None
    if inject_w is not None:
        w_list = [np.ascontiguousarray(w, dtype=np.float64) for w in inject_w]
        w_arr = (_dp * nrun)(*[dptr(w) for w in w_list])
    opts = OrRunOpts()
    opts.threads = threads
    ids = None
    if chain_ids is not None:
        ids = (C.c_size_t * nrun)(*chain_ids)
        opts.chain_ids = ids
        opts.n_ids = nrun
    st = oracle().or_run_ex(C.byref(cfg), C.byref(tgt), w_arr, C.byref(out), C.byref(opts))
    if st != 0:
        raise RuntimeError(f"oracle run failed {st}: {oracle().or_last_error().decode()}")
    n = out.batches
    res.update(batches=n, total_samples=out.total_samples, accumulated_samples=out.accumulated_samples,
               stop_reason=STOP[out.stop_reason], n_lag=nl)
    for key in ("cov_error_hist", "mean_error_hist", "psrf_hist"):
        res[key] = res[key][:n]
    res["beta_hist"] = res["beta_hist"][:, : n * M]
    res["acc_hist"] = res["acc_hist"][:, : n * M]
    if traces:
        res["traces"] = res["traces"][:, :, : out.trace_len]
    return res
