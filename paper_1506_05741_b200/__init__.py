"""paper_1506_05741_b200 — B200-native DIAM sampler hot path.

The product is ``libdiam.so`` in this directory: the reference's ``diam.h`` C
ABI (proj/include/diam/diam.h) implemented by a C++ engine over hand-written
sm_100a kernels (csrc/). Python here is a binding for tests and benchmarks,
not a second implementation: there is no CPU fallback, and loading fails
loudly when the library has not been built.
"""
from __future__ import annotations

import ctypes as C
import os

from .abi import DiamABI, DiamError, RunOptions  # noqa: F401

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(PKG_DIR, "libdiam.so")

_abi = None


def lib_path() -> str:
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(
            f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
            "(make -C paper_1506_05741_b200/csrc). There is no CPU fallback.")
    return LIB_PATH


def load() -> "B200":
    """Load the B200 libdiam.so (once per process)."""
    global _abi
    if _abi is None:
        _abi = B200(lib_path())
    return _abi


_vp = C.c_void_p
_dp = C.POINTER(C.c_double)


class B200(DiamABI):
    """diam.h plus the diam_b200.h extensions (include/diam_b200.h)."""

    def __init__(self, path: str):
        super().__init__(path)
        L = self.lib
        st, i64, u64 = C.c_int, C.c_int64, C.c_uint64
        spec = {
            "diamx_build_info": (C.c_char_p, []),
            "diamx_launch_count": (u64, []),
            "diamx_fp64_peak": (st, [_dp]),
            "diamx_nccl_unique_id": (st, [C.c_char_p]),
            "diamx_comm_init": (st, [C.c_char_p, C.c_int, C.c_int]),
            "diamx_comm_destroy": (None, []),
            "diamx_comm_size": (st, [C.POINTER(C.c_int)]),
            "diamx_engine_create": (st, [_vp, C.POINTER(RunOptions), C.POINTER(_vp)]),
            "diamx_engine_run_batches": (st, [_vp, i64, _dp]),
            "diamx_engine_set_profiling": (st, [_vp, C.c_int]),
            "diamx_engine_stat": (st, [_vp, C.c_char_p, _dp, _dp, C.POINTER(i64)]),
            "diamx_engine_flops_per_batch": (C.c_double, [_vp]),
            "diamx_engine_local_chains": (i64, [_vp]),
            "diamx_engine_layout": (st, [_vp, C.POINTER(i64), C.POINTER(i64), C.POINTER(i64)]),
            "diamx_engine_free": (None, [_vp]),
            "diamx_sample_capture": (st, [_vp, C.POINTER(RunOptions), C.POINTER(_vp), C.POINTER(_vp)]),
            "diamx_sample_threads": (st, [_vp, C.POINTER(RunOptions), C.c_int, C.POINTER(_vp)]),
            "diamx_resume_threads": (st, [C.c_char_p, C.POINTER(RunOptions), C.c_int, C.POINTER(_vp)]),
            "diamx_capture_len": (i64, [_vp, i64, C.c_char_p]),
            "diamx_capture_copy": (st, [_vp, i64, C.c_char_p, _dp, i64]),
            "diamx_draws": (st, [C.c_int, _vp, _vp, i64, u64, u64, C.c_char_p, u64, _vp]),
            "diamx_gemm": (st, [_vp, _vp, _vp, C.c_int, C.c_int, C.c_int, i64, i64, i64, C.c_int, C.c_int,
                                C.c_double, C.c_double, C.c_int, C.c_int, _vp]),
            "diamx_potrf": (st, [_vp, i64, i64, C.c_int, C.c_int, _vp, _vp]),
            "diamx_trsv": (st, [_vp, i64, i64, _vp, _vp, _vp, C.c_int, C.c_int, _vp]),
            "diamx_potrf_bench": (st, [_vp, i64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _dp]),
        }
        for name, (res, args) in spec.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args

    # -------------------------------------------------------------- engine
    def engine(self, target, **opts) -> "Engine":
        o = self.options(**opts)
        h = C.c_void_p()
        self.check(self.lib.diamx_engine_create(target.h, C.byref(o), C.byref(h)))
        return Engine(self, h)

    def sample_capture(self, target, **opts):
        from .abi import Result
        o = self.options(**opts)
        r, e = C.c_void_p(), C.c_void_p()
        self.check(self.lib.diamx_sample_capture(target.h, C.byref(o), C.byref(r), C.byref(e)))
        return Result(self, r), Capture(self, e)

    def sample_threads(self, target, world: int, **opts):
        """The sharded engine path (`world` ranks) on one GPU, in-process exchange."""
        from .abi import Result
        o = self.options(**opts)
        r = C.c_void_p()
        self.check(self.lib.diamx_sample_threads(target.h, C.byref(o), world, C.byref(r)))
        return Result(self, r)

    def resume_threads(self, path: str, world: int, overrides=None):
        """diam_resume with `world` in-process ranks (the sharded restore)."""
        from .abi import Result
        r = C.c_void_p()
        self.check(self.lib.diamx_resume_threads(path.encode(), C.byref(overrides) if overrides else None, world,
                                                 C.byref(r)))
        return Result(self, r)

    def launch_count(self) -> int:
        return int(self.lib.diamx_launch_count())


class Engine:
    def __init__(self, abi: B200, h):
        self.abi, self.h = abi, h

    def __del__(self):
        try:
            self.abi.lib.diamx_engine_free(self.h)
        except Exception:
            pass

    def run_batches(self, k: int) -> float:
        ms = C.c_double()
        self.abi.check(self.abi.lib.diamx_engine_run_batches(self.h, k, C.byref(ms)))
        return ms.value

    def set_profiling(self, on: bool) -> None:
        self.abi.check(self.abi.lib.diamx_engine_set_profiling(self.h, int(on)))

    def stat(self, name: str):
        ms, fl, n = C.c_double(), C.c_double(), C.c_int64()
        self.abi.check(self.abi.lib.diamx_engine_stat(self.h, name.encode(), C.byref(ms), C.byref(fl), C.byref(n)))
        return ms.value, fl.value, n.value

    @property
    def flops_per_batch(self) -> float:
        return self.abi.lib.diamx_engine_flops_per_batch(self.h)

    @property
    def local_chains(self) -> int:
        return self.abi.lib.diamx_engine_local_chains(self.h)

    @property
    def layout(self) -> dict:
        g, lc, pf = C.c_int64(), C.c_int64(), C.c_int64()
        self.abi.check(self.abi.lib.diamx_engine_layout(self.h, C.byref(g), C.byref(lc), C.byref(pf)))
        return {"groups": g.value, "chunk_rows": lc.value, "pool_factors": pf.value}


class Capture(Engine):
    def get(self, chain: int, which: str):
        import numpy as np
        n = self.abi.lib.diamx_capture_len(self.h, chain, which.encode())
        if n < 0:
            raise IndexError(which)
        out = np.zeros(max(n, 1))
        self.abi.check(self.abi.lib.diamx_capture_copy(self.h, chain, which.encode(),
                                                       out.ctypes.data_as(_dp), out.size))
        return out[:n]
