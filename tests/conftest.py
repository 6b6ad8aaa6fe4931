import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    # build the product library and the oracle if they are missing (no-op when built)
    for d in ("paper_1102_2878_b200", "oracle"):
        path = os.path.join(ROOT, d)
        if os.path.exists(os.path.join(path, "Makefile")):
            subprocess.run(["make", "-s", "-C", path], check=False,
                           stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)


def _has_gpu():
    try:
        import ctypes
        lib = ctypes.CDLL(os.path.join(ROOT, "paper_1102_2878_b200", "libdfgtb.so"))
        return lib.dfgtb_device_count() > 0
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _has_gpu():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    from oracle import load_oracle
    return load_oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import load_reference
    r = load_reference()
    if r is None:
        pytest.skip("compiled reference (oracle/_ref/libdfgt_ref.so) not available")
    return r


@pytest.fixture(scope="session")
def dfgtb():
    import paper_1102_2878_b200 as m
    return m
