"""Host-side helpers of the product vs the reference (no GPU needed).

pilot_bandwidth (cv.cpp:112-139) in both host mirrors -- the Python package
(engine.py) and the C++ header (include/dfgtb.hpp) -- must be bit-identical to the
reference's: the same two-pass sequential sums, the same pow.
"""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _sets():
    from paper_1102_2878_b200 import datagen
    g = np.random.default_rng(12)
    return [datagen.uniform(10_000, 2, 1001), datagen.gauss_mixture_2d(20_000, 3),
            datagen.clustered_3d(5000, 4), datagen.full_cov_mixture_5d(3000, 5),
            g.normal(size=(7, 1)) * 1e8 + 3.0, g.random((2, 6))]


def test_python_pilot_bandwidth_bit_exact(orc):
    import paper_1102_2878_b200 as dfgtb
    for x in _sets():
        assert dfgtb.pilot_bandwidth(x) == orc.pilot_bandwidth(x)


def test_python_pilot_bandwidth_vs_compiled_reference(ref):
    import paper_1102_2878_b200 as dfgtb
    for x in _sets():
        assert dfgtb.pilot_bandwidth(x) == ref.pilot_bandwidth(x)
    with pytest.raises(ValueError, match="at least 2 points"):
        dfgtb.pilot_bandwidth(np.zeros((1, 2)))
    with pytest.raises(ValueError, match="zero-variance"):
        dfgtb.pilot_bandwidth(np.ones((5, 2)))


def test_cpp_header_pilot_bandwidth_bit_exact(orc, tmp_path):
    exe = tmp_path / "pilot"
    subprocess.run(["g++", "-std=c++20", "-O2", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "pilot_main.cpp"), "-o", str(exe)],
                   check=True)
    for i, x in enumerate(_sets() + [np.ones((4, 3))]):
        f = tmp_path / f"x{i}.bin"
        with open(f, "wb") as fh:
            fh.write(np.array(x.shape, np.uint64).tobytes())
            fh.write(np.ascontiguousarray(x, np.float64).tobytes())
        out = subprocess.run([str(exe), str(f)], check=True, capture_output=True, text=True).stdout.strip()
        if np.all(x == x[0]):
            assert out.startswith("invalid_argument: pilot bandwidth undefined")
        else:
            assert float(out) == orc.pilot_bandwidth(x), i
