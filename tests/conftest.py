import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")


@pytest.fixture(scope="session")
def b200():
    import paper_1506_05741_b200 as pkg
    return pkg.load()


@pytest.fixture(scope="session")
def ref_abi():
    import _oracle as O
    from paper_1506_05741_b200.abi import DiamABI
    if not O.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return DiamABI(O.REF_SO)


@pytest.fixture(scope="session")
def tmpdir_s(tmp_path_factory):
    return tmp_path_factory.mktemp("diam")


def has_cuda() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
