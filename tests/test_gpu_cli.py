"""The C++ host path: tools/dfgtb_cli.cpp (reference cli.cpp `kde` / `cv` semantics over
include/dfgtb.hpp -> the C ABI -> the GPU engine), driven through files like the
reference CLI, checked against the oracle."""
import os
import subprocess

import numpy as np
import pytest

from paper_1102_2878_b200 import datagen

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def cli(tmp_path_factory):
    out = str(tmp_path_factory.mktemp("cli") / "dfgtb_cli")
    lib = os.path.join(ROOT, "paper_1102_2878_b200")
    rc = subprocess.run(["g++", "-std=c++20", "-O1", f"-I{ROOT}/include",
                         os.path.join(ROOT, "tools", "dfgtb_cli.cpp"), "-o", out, f"-L{lib}",
                         "-ldfgtb", f"-Wl,-rpath,{lib}"], capture_output=True, text=True)
    assert rc.returncode == 0, rc.stderr
    return out


def _write(path, x, delim=","):
    with open(path, "w") as f:
        for row in x:
            f.write(delim.join(repr(float(v)) for v in row) + "\n")


def test_cli_kde_raw_sums_and_density(cli, orc, tmp_path):
    x = datagen.config(2, scale_n=0.03).refs
    h = 0.02
    _write(tmp_path / "r.csv", x)
    subprocess.run([cli, "kde", "--refs", str(tmp_path / "r.csv"), "--bandwidth", str(h),
                    "--out", str(tmp_path / "s.txt"), "--raw-sums", "--leaf-threshold", "32"],
                   check=True)
    got = np.loadtxt(tmp_path / "s.txt")
    exact = orc.naive_kde(x, x, h)
    assert np.max(np.abs(got - exact) / exact) <= 0.01
    # default output: densities G / (N (2 pi h^2)^(D/2)), whitespace input, Q != R
    q = np.random.default_rng(5).random((77, 2))
    _write(tmp_path / "r.txt", x, " ")
    _write(tmp_path / "q.txt", q, " ")
    subprocess.run([cli, "kde", "--refs", str(tmp_path / "r.txt"), "--queries", str(tmp_path / "q.txt"),
                    "--bandwidth", str(h), "--out", str(tmp_path / "d.txt")], check=True)
    dens = np.loadtxt(tmp_path / "d.txt")
    ex = orc.naive_kde(q, x, h) / (x.shape[0] * 2 * np.pi * h * h)
    ok = ex > 0
    assert np.max(np.abs(dens[ok] - ex[ok]) / ex[ok]) <= 0.01


def test_cli_cv_table(cli, orc, tmp_path):
    x = datagen.config(2, scale_n=0.03).refs
    _write(tmp_path / "r.csv", x)
    base = 0.02
    subprocess.run([cli, "cv", "--refs", str(tmp_path / "r.csv"), "--out", str(tmp_path / "t.csv"),
                    "--score", "lscv", "--scales", "0.5,1,2", "--base-h", str(base),
                    "--leaf-threshold", "32"], check=True)
    lines = open(tmp_path / "t.csv").read().strip().splitlines()
    assert lines[0] == "scale,h,score,seconds,max_rel_err"
    for line, s in zip(lines[1:], (0.5, 1.0, 2.0)):
        f = line.split(",")
        h = float(f[1])
        assert abs(h - s * base) <= 1e-12
        ex = orc.lscv(2, h, orc.naive_kde(x, x, h), 2 * h, orc.naive_kde(x, x, 2 * h))
        assert abs(float(f[2]) - ex) <= 0.05 * abs(ex)


def test_cli_errors(cli, tmp_path):
    r = subprocess.run([cli, "kde", "--refs", str(tmp_path / "missing.csv"), "--bandwidth", "0.1",
                        "--out", str(tmp_path / "o")], capture_output=True, text=True)
    assert r.returncode == 2 and "error" in r.stderr
    r = subprocess.run([cli, "bogus"], capture_output=True, text=True)
    assert r.returncode == 2
