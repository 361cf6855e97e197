"""The C ABI from plain C (-m gpu): examples/track_c.c -- a small tracking run
through phd_create / phd_set_particles / phd_step / phd_destroy, no Python in
the loop -- compiled against include/phd.h and libphd.so, run, and required to
track every target within 50 m and to refuse an out-of-order call."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_c_example_tracks_targets(tmp_path):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as phd
    phd.load()
    libdir = os.path.dirname(phd.lib_path())
    exe = str(tmp_path / "track_c")
    subprocess.run(["gcc", "-O2", "-I", os.path.join(ROOT, "include"), os.path.join(ROOT, "examples", "track_c.c"),
                    "-L", libdir, "-l:libphd.so", "-Wl,-rpath," + libdir, "-lm", "-o", exe], check=True)
    r = subprocess.run([exe], stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True, timeout=300)
    assert r.returncode == 0, r.stdout[-3000:]
    assert "out of order -> call out of order" in r.stdout  # PHD_ESTATE
