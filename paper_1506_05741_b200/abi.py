"""ctypes binding of the ``diam.h`` C ABI.

The same binding loads either implementation of the ABI:

* this package's ``libdiam.so`` (B200 engine, the product), or
* the reference's ``libdiam.so`` (proj/include/diam/diam.h, proj/src/capi.cpp),

because the two export the same 42 symbols with the same prototypes. This is
the ctypes stub a maintainer of a Python caller of the reference would add;
see INTEGRATION.md.
"""
from __future__ import annotations

import ctypes as C
import math
from typing import Optional

import numpy as np

_dp = C.POINTER(C.c_double)

STATUS = {
    0: "DIAM_OK", 1: "DIAM_ERR_INVALID_ARGUMENT", 2: "DIAM_ERR_INVALID_DIMENSION",
    3: "DIAM_ERR_DIMENSION_MISMATCH", 4: "DIAM_ERR_NOT_POSITIVE_DEFINITE",
    5: "DIAM_ERR_SINGULAR_DIAGONAL", 6: "DIAM_ERR_CONVERGENCE_FAILURE", 7: "DIAM_ERR_DEGENERATE_TRACE",
    8: "DIAM_ERR_ZERO_WITHIN_VARIANCE", 9: "DIAM_ERR_UNEQUAL_BATCH_SIZES", 10: "DIAM_ERR_IO",
    11: "DIAM_ERR_UNKNOWN",
}


class DiamError(RuntimeError):
    def __init__(self, status: int, message: str):
        super().__init__(f"{STATUS.get(status, status)}: {message}")
        self.status = status
        self.message = message


class RunOptions(C.Structure):
    """diam_run_options (proj/include/diam/diam.h:66-94)."""
    _fields_ = [
        ("kernel", C.c_char_p), ("beta_init", C.c_double), ("inflation", C.c_double),
        ("band_lo", C.c_double), ("band_hi", C.c_double), ("n_lag", C.c_int64), ("n0", C.c_int64),
        ("n_ref_start", C.c_int64), ("adaptive_ref", C.c_int), ("use_explicit_inverse", C.c_int),
        ("adapt_beta", C.c_int), ("chains", C.c_int64), ("intervals_per_batch", C.c_int64),
        ("max_batches", C.c_int64), ("cov_tol", C.c_double), ("mean_tol", C.c_double),
        ("psrf_tol", C.c_double), ("max_samples", C.c_int64), ("max_wall_seconds", C.c_double),
        ("init_dispersion", C.c_double), ("master_seed", C.c_uint64), ("record_traces", C.c_int),
        ("trace_thin", C.c_int64), ("trace_eigen_projections", C.c_int),
        ("checkpoint_path", C.c_char_p), ("threads", C.c_int64),
    ]


def _proto(lib, name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)


class DiamABI:
    """Thin object wrapper over one loaded implementation of diam.h."""

    def __init__(self, path: str, mode: int = C.RTLD_LOCAL):
        self.path = path
        self.lib = L = C.CDLL(path, mode=mode)
        vp, i64, u64, st = C.c_void_p, C.c_int64, C.c_uint64, C.c_int
        _proto(L, "diam_status_string", C.c_char_p, st)
        _proto(L, "diam_last_error", C.c_char_p)
        _proto(L, "diam_target_build", st, C.c_char_p, i64, u64, C.c_double, C.c_double, C.POINTER(vp))
        _proto(L, "diam_target_save", st, vp, C.c_char_p)
        _proto(L, "diam_target_load", st, C.c_char_p, C.POINTER(vp))
        _proto(L, "diam_target_free", None, vp)
        _proto(L, "diam_target_dim", i64, vp)
        _proto(L, "diam_target_seed", u64, vp)
        _proto(L, "diam_target_kind", C.c_char_p, vp)
        _proto(L, "diam_target_log_density", st, vp, _dp, i64, _dp)
        _proto(L, "diam_target_condition_number", st, vp, _dp)
        _proto(L, "diam_target_eigen_range", st, vp, _dp, _dp)
        _proto(L, "diam_target_analytic_mean", st, vp, _dp, i64)
        _proto(L, "diam_target_analytic_cov", st, vp, _dp, i64)
        _proto(L, "diam_run_options_init", None, C.POINTER(RunOptions))
        _proto(L, "diam_sample", st, vp, C.POINTER(RunOptions), C.POINTER(vp))
        _proto(L, "diam_resume", st, C.c_char_p, C.POINTER(RunOptions), C.POINTER(vp))
        _proto(L, "diam_result_free", None, vp)
        _proto(L, "diam_result_total_samples", u64, vp)
        _proto(L, "diam_result_accumulated_samples", u64, vp)
        _proto(L, "diam_result_batches", i64, vp)
        _proto(L, "diam_result_chains", i64, vp)
        _proto(L, "diam_result_dim", i64, vp)
        _proto(L, "diam_result_wall_seconds", C.c_double, vp)
        _proto(L, "diam_result_stop_reason", C.c_char_p, vp)
        _proto(L, "diam_result_final_cov_error", C.c_double, vp)
        _proto(L, "diam_result_final_mean_error", C.c_double, vp)
        _proto(L, "diam_result_final_max_psrf", C.c_double, vp)
        _proto(L, "diam_result_write_json", st, vp, C.c_char_p)
        _proto(L, "diam_result_copy_mean", st, vp, _dp, i64)
        _proto(L, "diam_result_copy_cov", st, vp, _dp, i64)
        _proto(L, "diam_result_copy_history", st, vp, C.c_char_p, _dp, i64)
        _proto(L, "diam_result_lag_boundaries", i64, vp, i64)
        _proto(L, "diam_result_copy_chain_history", st, vp, i64, C.c_char_p, _dp, i64)
        _proto(L, "diam_result_num_functionals", i64, vp)
        _proto(L, "diam_result_functional_name", C.c_char_p, vp, i64)
        _proto(L, "diam_result_trace_length", i64, vp, i64, i64)
        _proto(L, "diam_result_copy_trace", st, vp, i64, i64, _dp, i64)
        _proto(L, "diam_acf", st, _dp, i64, i64, _dp)
        _proto(L, "diam_iact", st, _dp, i64, _dp)
        _proto(L, "diam_ess", st, _dp, i64, _dp)
        _proto(L, "diam_fit_quadratic", st, _dp, _dp, i64, _dp, _dp, _dp)

    # ------------------------------------------------------------------ util
    def check(self, status: int) -> None:
        if status != 0:
            raise DiamError(status, self.lib.diam_last_error().decode())

    def options(self, **kw) -> RunOptions:
        o = RunOptions()
        self.lib.diam_run_options_init(C.byref(o))
        for k, v in kw.items():
            if k in ("kernel", "checkpoint_path") and isinstance(v, str):
                v = v.encode()
            setattr(o, k, v)
        return o

    # --------------------------------------------------------------- targets
    def target_build(self, kind: str, dim: int, seed: int, sigma2: float = 0.0, twist_b: float = -1.0):
        h = C.c_void_p()
        self.check(self.lib.diam_target_build(kind.encode(), dim, seed, sigma2, twist_b, C.byref(h)))
        return Target(self, h)

    def target_load(self, path: str):
        h = C.c_void_p()
        self.check(self.lib.diam_target_load(path.encode(), C.byref(h)))
        return Target(self, h)

    # ------------------------------------------------------------------ runs
    def sample(self, target: "Target", options: Optional[RunOptions] = None, **kw) -> "Result":
        o = options if options is not None else self.options(**kw)
        h = C.c_void_p()
        self.check(self.lib.diam_sample(target.h, C.byref(o), C.byref(h)))
        return Result(self, h)

    def resume(self, path: str, overrides: Optional[RunOptions] = None) -> "Result":
        h = C.c_void_p()
        self.check(self.lib.diam_resume(path.encode(), C.byref(overrides) if overrides else None,
                                        C.byref(h)))
        return Result(self, h)

    # ----------------------------------------------------------- diagnostics
    def iact(self, trace: np.ndarray) -> float:
        t = np.ascontiguousarray(trace, dtype=np.float64)
        out = C.c_double()
        self.check(self.lib.diam_iact(t.ctypes.data_as(_dp), t.size, C.byref(out)))
        return out.value

    def ess(self, trace: np.ndarray) -> float:
        t = np.ascontiguousarray(trace, dtype=np.float64)
        out = C.c_double()
        self.check(self.lib.diam_ess(t.ctypes.data_as(_dp), t.size, C.byref(out)))
        return out.value


class Target:
    def __init__(self, abi: DiamABI, h: C.c_void_p):
        self.abi, self.h = abi, h

    def __del__(self):
        try:
            self.abi.lib.diam_target_free(self.h)
        except Exception:
            pass

    @property
    def dim(self) -> int:
        return self.abi.lib.diam_target_dim(self.h)

    @property
    def kind(self) -> str:
        return self.abi.lib.diam_target_kind(self.h).decode()

    def save(self, path: str) -> None:
        self.abi.check(self.abi.lib.diam_target_save(self.h, path.encode()))

    def log_density(self, x: np.ndarray) -> float:
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = C.c_double()
        self.abi.check(self.abi.lib.diam_target_log_density(self.h, x.ctypes.data_as(_dp), x.size,
                                                            C.byref(out)))
        return out.value

    def analytic_cov(self) -> np.ndarray:
        d = self.dim
        out = np.zeros((d, d))
        self.abi.check(self.abi.lib.diam_target_analytic_cov(self.h, out.ctypes.data_as(_dp), d * d))
        return out

    def analytic_mean(self) -> np.ndarray:
        out = np.zeros(self.dim)
        self.abi.check(self.abi.lib.diam_target_analytic_mean(self.h, out.ctypes.data_as(_dp), out.size))
        return out


class Result:
    def __init__(self, abi: DiamABI, h: C.c_void_p):
        self.abi, self.h = abi, h

    def __del__(self):
        try:
            self.abi.lib.diam_result_free(self.h)
        except Exception:
            pass

    def _get(self, name):
        return getattr(self.abi.lib, "diam_result_" + name)(self.h)

    total_samples = property(lambda s: s._get("total_samples"))
    accumulated_samples = property(lambda s: s._get("accumulated_samples"))
    batches = property(lambda s: s._get("batches"))
    chains = property(lambda s: s._get("chains"))
    dim = property(lambda s: s._get("dim"))
    wall_seconds = property(lambda s: s._get("wall_seconds"))
    stop_reason = property(lambda s: s._get("stop_reason").decode())
    final_cov_error = property(lambda s: s._get("final_cov_error"))
    final_mean_error = property(lambda s: s._get("final_mean_error"))
    final_max_psrf = property(lambda s: s._get("final_max_psrf"))

    def mean(self) -> np.ndarray:
        out = np.zeros(self.dim)
        self.abi.check(self.abi.lib.diam_result_copy_mean(self.h, out.ctypes.data_as(_dp), out.size))
        return out

    def cov(self) -> np.ndarray:
        d = self.dim
        out = np.zeros((d, d))
        self.abi.check(self.abi.lib.diam_result_copy_cov(self.h, out.ctypes.data_as(_dp), d * d))
        return out

    def history(self, which: str) -> np.ndarray:
        out = np.zeros(max(self.batches, 1))
        self.abi.check(self.abi.lib.diam_result_copy_history(self.h, which.encode(),
                                                             out.ctypes.data_as(_dp), out.size))
        return out[: self.batches]

    def chain_history(self, chain: int, which: str) -> np.ndarray:
        n = self.abi.lib.diam_result_lag_boundaries(self.h, chain)
        out = np.zeros(max(n, 1))
        self.abi.check(self.abi.lib.diam_result_copy_chain_history(self.h, chain, which.encode(),
                                                                   out.ctypes.data_as(_dp), out.size))
        return out[:n]

    def functional_names(self):
        n = self.abi.lib.diam_result_num_functionals(self.h)
        return [self.abi.lib.diam_result_functional_name(self.h, i).decode() for i in range(n)]

    def trace(self, chain: int, functional: int) -> np.ndarray:
        n = self.abi.lib.diam_result_trace_length(self.h, chain, functional)
        if n < 0:
            raise IndexError("no such trace")
        out = np.zeros(max(n, 1))
        self.abi.check(self.abi.lib.diam_result_copy_trace(self.h, chain, functional,
                                                           out.ctypes.data_as(_dp), out.size))
        return out[:n]

    def write_json(self, path: str) -> None:
        self.abi.check(self.abi.lib.diam_result_write_json(self.h, path.encode()))


def finite(v: float) -> bool:
    return math.isfinite(v)
