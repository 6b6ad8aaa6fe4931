"""C-ABI checks that need no GPU: libdfgtb.so loads, exports every symbol that
include/dfgtb.h declares, host-side CV reductions match the oracle, and invalid
arguments fail with the reference's invalid_argument code before touching CUDA."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "dfgtb.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dfgtb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    from paper_1102_2878_b200 import _capi
    names = _declared()
    assert len(names) >= 20
    for n in names:
        assert hasattr(_capi.lib, n), n
    assert set(names) == set(_capi.EXPORTS)


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1102_2878_b200", "libdfgtb.so")
    out = os.popen(f"cuobjdump --list-elf {so} 2>/dev/null").read()
    if not out:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out
    assert all("sm_100a" in line for line in out.splitlines() if ".cubin" in line)


def test_host_cv_reductions_match_oracle(orc):
    from paper_1102_2878_b200 import lkcv_from_sums, lscv_from_sums
    rng = np.random.default_rng(0)
    refs = rng.random((1000, 2))
    s1 = 1.0 + 50.0 * rng.random(1000)
    s1[:7] = 0.999  # clamped leave-one-out sums
    s2 = 1.0 + 80.0 * rng.random(1000)
    r = lkcv_from_sums(refs, 0.05, s1)
    lk, cl = orc.lkcv(2, 0.05, s1)
    assert r.score == lk and r.clamped == cl == 7
    assert lscv_from_sums(refs, 0.05, s1, 0.1, s2).score == pytest.approx(
        orc.lscv(2, 0.05, s1, 0.1, s2), rel=1e-14)


def test_invalid_arguments_before_cuda():
    import paper_1102_2878_b200 as m
    x = np.random.default_rng(1).random((20, 2))
    with pytest.raises(ValueError, match="epsilon"):
        m.DualTreeEngine(x, config=m.EngineConfig(epsilon=-0.5))
    with pytest.raises(ValueError, match="leaf_threshold"):
        m.DualTreeEngine(x, config=m.EngineConfig(leaf_threshold=0))
    with pytest.raises(ValueError, match="p_max"):
        m.DualTreeEngine(x, config=m.EngineConfig(p_max=16))
    with pytest.raises(ValueError):
        m.DualTreeEngine(np.zeros((0, 2)))
    with pytest.raises(ValueError):
        m.lkcv_from_sums(np.zeros((1, 2)), 0.1, np.ones(1))
    with pytest.raises(ValueError):
        m.gaussian_normalizer(2, 0.0)
    with pytest.raises(ValueError):
        m.verify_relative_error([1.0], [0.0])


def test_verify_relative_error_basics():
    import paper_1102_2878_b200 as m
    e = [1.0, 2.0, 4.0]
    assert m.verify_relative_error(e, e).max_relative_error == 0.0
    r = m.verify_relative_error([1.0, 2.2, 4.0], e)
    assert r.worst_index == 1 and r.max_relative_error == pytest.approx(0.1)


def test_device_count_never_raises():
    from paper_1102_2878_b200 import _capi
    assert _capi.lib.dfgtb_device_count() >= 0


def test_cpp_header_shim_compiles():
    """include/dfgtb.hpp (the C++ mirror of dfgt::DualTreeEngine etc.) compiles and
    links against the C ABI."""
    hpp = os.path.join(ROOT, "include", "dfgtb.hpp")
    if not os.path.exists(hpp):
        pytest.skip("no C++ shim")
    src = os.path.join(ROOT, "tools", "dfgtb_cli.cpp")
    out = "/tmp/dfgtb_cli_test"
    rc = os.system(f"g++ -std=c++20 -O1 -I{ROOT}/include {src} -o {out} "
                   f"-L{ROOT}/paper_1102_2878_b200 -ldfgtb -Wl,-rpath,{ROOT}/paper_1102_2878_b200")
    assert rc == 0
