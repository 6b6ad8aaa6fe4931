"""Memory-safety workload: run under compute-sanitizer (tools/sanitize.sh, where the pool
allows it) or with DFGTB_GUARD=1, where every phase is followed by dfgtb_guard_check()
(guard bands past every device block; tests/test_gpu_guard.py).  smoke(), then a config-2
sweep at 5% of N on FRESH engines (the first batch of an engine runs with optimistic
buffers and overflows -> the host regrows and reruns it), a Q != R batch, the FP64-only
base case, the L2L chain and the DFD mode -- every kernel family of the product path.

  python tools/sanitize_run.py [--small]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402


def main():
    small = "--small" in sys.argv
    import __graft_entry__ as g
    import paper_1102_2878_b200 as dfgtb
    from paper_1102_2878_b200 import _capi, datagen

    guard = os.environ.get("DFGTB_GUARD") is not None
    import builtins
    _print = builtins.print

    def print(*a):  # noqa: A001 -- every phase line is followed by the guard verdict
        _print(*a, flush=True)
        if guard:
            bad = _capi.lib.dfgtb_guard_check()
            _print(f"  guard bands written: {bad}", flush=True)
            if bad != 0:
                raise SystemExit(f"out-of-bounds write detected after: {a[0]}")

    if guard:
        if _capi.lib.dfgtb_guard_selftest() != 1:
            raise SystemExit("guard self-test did not detect its own out-of-bounds write")
        print("guard self-test ok")
    g.smoke()
    print("smoke ok")
    n = 1000 if small else 2500  # 5% of cfg2's 50k
    x = datagen.gauss_mixture_2d(n, seed=7)
    hs = float(dfgtb.pilot_bandwidth(x))
    scales = [1e-3, 1e-2, 1e-1, 10 ** -0.5, 1.0, 10 ** 0.5, 10.0, 100.0, 1000.0]
    cfg = dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32)
    with dfgtb.DualTreeEngine(x, dfgtb.Mode.series, cfg) as e:
        rows = e.sweep(scales, hs)
        rows = e.sweep(scales, hs)  # second batch: buffers sized from the first
        print("sweep ok", [round(r.ls_score, 6) for r in rows][:3])
    rng = np.random.default_rng(11)
    q = rng.random((n // 2, 2))
    with dfgtb.DualTreeEngine(x, dfgtb.Mode.series, cfg) as e:
        s = e.compute_batch(q, [hs * 0.1, hs, hs * 10])
        print("Q != R ok", float(s.sum()))
    os.environ["DFGTB_NO_F32"] = "1"
    try:
        with dfgtb.DualTreeEngine(x, dfgtb.Mode.series, cfg) as e:
            print("no-f32 ok", float(e.compute(None, hs * 0.01).sum()))
    finally:
        del os.environ["DFGTB_NO_F32"]
    x3 = rng.random((n, 3))
    with dfgtb.DualTreeEngine(x3, dfgtb.Mode.series, dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32,
                                                                      local_pushdown=1)) as e:
        print("3-D L2L ok", float(e.compute(None, 0.05).sum()))
    x5 = rng.random((n // 2, 5))
    with dfgtb.DualTreeEngine(x5, dfgtb.Mode.series, dfgtb.EngineConfig(epsilon=0.01, leaf_threshold=32,
                                                                      p_max=4)) as e:
        print("5-D p4 ok", float(e.compute(None, 0.2).sum()))
    with dfgtb.DualTreeEngine(x, dfgtb.Mode.centroid, cfg) as e:
        print("DFD ok", float(e.compute(None, hs).sum()))
    print("sanitize workload done")


if __name__ == "__main__":
    main()
