"""Device bounds checks (-m gpu): the library rebuilt with -DPHD_DEBUG_BOUNDS
(PHD_DCHECK in the kernels traps on an out-of-range index) runs
tools/bounds_case.py -- every kernel, both sensors, the gated path with
multi-chunk tiles and M > 4096 -- in a subprocess.  compute-sanitizer is not
available on the GPU pool, so these checks stand in for memcheck."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_debug_bounds_build_runs_clean():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    sys.path.insert(0, ROOT)
    from paper_1503_03769_b200 import build
    lib = os.path.join(ROOT, "paper_1503_03769_b200", "lib_variants", "debug.so")
    build.build(out=lib, extra=["-DPHD_DEBUG_BOUNDS"])
    env = dict(os.environ, PHD_LIB=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "bounds_case.py")], env=env, cwd=ROOT,
                       stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=900)
    assert r.returncode == 0 and "case done" in r.stdout, r.stdout[-3000:]
    assert "PHD_DCHECK failed" not in r.stdout
