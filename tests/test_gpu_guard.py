"""Out-of-bounds write check of the whole product path (compute-sanitizer is closed on
this pool): with DFGTB_GUARD=1 every device block carries a 4 KB guard band past its end;
tools/sanitize_run.py runs smoke(), a config-2 sweep at 5% N on fresh engines (first
batches overflow their optimistic buffers and rerun), Q != R batches, the FP64-only base
case, the L2L chain at D = 3, 5-D p_max = 4 and the DFD mode, and checks after every
phase that no band was written.  The guard's own self-test (one element written past a
block) must be caught first."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("tiny", [False, True])
def test_no_out_of_bounds_writes(tiny):
    """tiny: DFGTB_TINY_CAPS starts every traversal buffer at 64 elements, so every first
    batch overflows, regrows and reruns several times."""
    env = dict(os.environ, DFGTB_GUARD="1")
    if tiny:
        env["DFGTB_TINY_CAPS"] = "1"
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sanitize_run.py"), "--small"],
                         env=env, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "guard self-test ok" in out.stdout
    assert "sanitize workload done" in out.stdout
    assert out.stdout.count("guard bands written: 0") >= 8, out.stdout
