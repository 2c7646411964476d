"""CPU-side checks of the drop-in boundary (no GPU compute).

* libdiam.so loads and exports every symbol include/diam/diam.h and
  include/diam_b200.h declare;
* host-side ABI functions match the reference bit-for-bit: target
  construction (DIAMTGT bytes), log density, acf/iact/ess, quadratic fit,
  status strings, sentinel defaults, error codes and capacity checks
  (proj/src/capi.cpp, proj/tests/test_capi.cpp).
"""
import ctypes as C
import filecmp
import os
import re

import numpy as np
import pytest

from conftest import ROOT, has_cuda
from paper_1506_05741_b200.abi import DiamError

HEADERS = [os.path.join(ROOT, "include", "diam", "diam.h"), os.path.join(ROOT, "include", "diam_b200.h")]


def declared_symbols():
    names = set()
    for h in HEADERS:
        txt = open(h).read()
        txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
        for m in re.finditer(r"\b(diamx?_[a-z0-9_]+)\s*\(", txt):
            names.add(m.group(1))
    return names


def test_exports_every_declared_symbol(b200):
    syms = declared_symbols()
    assert len([s for s in syms if s.startswith("diam_")]) == 42
    for s in sorted(syms):
        assert hasattr(b200.lib, s), s


def test_same_diam_symbols_as_reference(b200, ref_abi):
    import subprocess
    def dyn(path):
        out = subprocess.run(["nm", "-D", "--defined-only", path], capture_output=True, text=True).stdout
        return {l.split()[-1] for l in out.splitlines() if re.search(r" T diam_", l)}
    assert dyn(b200.path) == dyn(ref_abi.path)


@pytest.mark.parametrize("kind,d", [("pi1", 24), ("pi2", 17), ("pi3", 30), ("pi4", 20), ("pi5", 40), ("pi6", 20)])
def test_target_build_bit_exact(b200, ref_abi, tmp_path, kind, d):
    a = ref_abi.target_build(kind, d, 9)
    b = b200.target_build(kind, d, 9)
    pa, pb = str(tmp_path / "a.bin"), str(tmp_path / "b.bin")
    a.save(pa)
    b.save(pb)
    assert filecmp.cmp(pa, pb, shallow=False)
    x = np.random.default_rng(d).normal(size=d) * 2
    assert a.log_density(x) == b.log_density(x)
    assert a.log_density(np.zeros(d)) == 0.0 == b.log_density(np.zeros(d))


def test_target_load_roundtrip(b200, tmp_path):
    t = b200.target_build("pi1", 12, 3)
    p = str(tmp_path / "t.bin")
    t.save(p)
    u = b200.target_load(p)
    assert u.dim == 12 and u.kind == "pi1"
    assert np.array_equal(t.analytic_cov(), u.analytic_cov())


def test_error_codes_and_messages(b200):
    with pytest.raises(DiamError) as e:
        b200.target_build("pi1", 1, 0)
    assert e.value.status == 2
    with pytest.raises(DiamError) as e:
        b200.target_build("pi5", 30, 0)
    assert e.value.status == 2 and "divisible by 20" in e.value.message
    with pytest.raises(DiamError) as e:
        b200.target_build("nope", 10, 0)
    assert e.value.status == 1
    with pytest.raises(DiamError) as e:
        b200.target_load("/nonexistent/x.bin")
    assert e.value.status == 10
    t = b200.target_build("pi1", 4, 1)
    with pytest.raises(DiamError) as e:
        t.log_density(np.zeros(3))
    assert e.value.status == 3
    # capacity check
    out = np.zeros(3)
    st = b200.lib.diam_target_analytic_mean(t.h, out.ctypes.data_as(C.POINTER(C.c_double)), 3)
    assert st == 1 and b"too small" in b200.lib.diam_last_error()
    # success clears the message
    t.log_density(np.zeros(4))
    assert b200.lib.diam_last_error() == b""
    for s in range(12):
        assert b200.lib.diam_status_string(s) == b200.lib.diam_status_string(s)
    assert b200.lib.diam_status_string(99) == b"unknown error"


def test_status_strings_match_reference(b200, ref_abi):
    for s in list(range(12)) + [42]:
        assert b200.lib.diam_status_string(s) == ref_abi.lib.diam_status_string(s)


def test_options_init_matches_reference(b200, ref_abi):
    a, b = b200.options(), ref_abi.options()
    for name, _ in a._fields_:
        assert getattr(a, name) == getattr(b, name), name


def test_diagnostics_match_reference(b200, ref_abi):
    rng = np.random.default_rng(0)
    x = np.zeros(5000)
    for i in range(1, x.size):
        x[i] = 0.9 * x[i - 1] + rng.normal()
    assert b200.iact(x) == ref_abi.iact(x)
    assert b200.ess(x) == ref_abi.ess(x)
    rho_a, rho_b = np.zeros(11), np.zeros(11)
    dp = C.POINTER(C.c_double)
    for lib, rho in ((b200.lib, rho_a), (ref_abi.lib, rho_b)):
        assert lib.diam_acf(x.ctypes.data_as(dp), x.size, 10, rho.ctypes.data_as(dp)) == 0
    assert np.array_equal(rho_a, rho_b)
    xs = np.linspace(100, 1000, 7)
    ys = 3 + 0.1 * xs + 2e-4 * xs ** 2 + rng.normal(size=7)
    res = []
    for lib in (b200.lib, ref_abi.lib):
        co, qs, rss = np.zeros(3), C.c_double(), C.c_double()
        assert lib.diam_fit_quadratic(xs.ctypes.data_as(dp), ys.ctypes.data_as(dp), 7, co.ctypes.data_as(dp),
                                      C.byref(qs), C.byref(rss)) == 0
        res.append((list(co), qs.value, rss.value))
    assert res[0] == res[1]
    # degenerate trace -> DIAM_ERR_DEGENERATE_TRACE on both
    c = np.ones(100)
    out = C.c_double()
    assert b200.lib.diam_iact(c.ctypes.data_as(dp), 100, C.byref(out)) == 7
    assert ref_abi.lib.diam_iact(c.ctypes.data_as(dp), 100, C.byref(out)) == 7


def test_resume_rejects_missing_and_foreign_files(b200, tmp_path):
    with pytest.raises(DiamError) as e:
        b200.resume(str(tmp_path / "missing.ckpt"))
    assert e.value.status == 10
    t = b200.target_build("pi1", 4, 1)
    p = str(tmp_path / "target.bin")
    t.save(p)  # a DIAMTGT file is not a DIAMCKPT file
    with pytest.raises(DiamError) as e:
        b200.resume(p)
    assert e.value.status == 10 and "not a checkpoint" in e.value.message


@pytest.mark.skipif(has_cuda(), reason="checks the no-GPU failure path")
def test_no_cpu_fallback(b200):
    t = b200.target_build("pi1", 4, 1)
    with pytest.raises(DiamError) as e:
        b200.sample(t, chains=1, max_batches=1)
    assert "CUDA" in e.value.message
