"""Device Philox known-answer test (the noise of Eq 5):
the kernels' Philox4x32-10 (phd_philox4x32_10_device) against cuRAND's
curand_Philox4x32_10 on 10^6 counters -- the filter's counter layouts (slot, step,
stream, slot >> 32) for streams 1-5 plus random 128-bit counters -- and, on a sample,
against the host build (itself pinned to ATen's philox_engine), -m gpu."""
import os
import subprocess

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))


def _counters(n, seed):
    rng = np.random.default_rng(seed)
    c = np.empty((n, 4), np.uint32)
    m = n // 2
    g = rng.integers(0, 2**34, m, dtype=np.uint64)  # filter layout: (g lo, k, stream, g hi)
    c[:m, 0] = (g & 0xFFFFFFFF).astype(np.uint32)
    c[:m, 1] = rng.integers(0, 200, m).astype(np.uint32)
    c[:m, 2] = rng.integers(1, 6, m).astype(np.uint32)
    c[:m, 3] = (g >> 32).astype(np.uint32)
    c[m:] = rng.integers(0, 2**32, (n - m, 4), dtype=np.uint64).astype(np.uint32)
    c[m] = 0
    c[m + 1] = 0xFFFFFFFF
    return c


@pytest.mark.parametrize("seed", [1, 0x123456789ABCDEF0])
def test_device_philox_matches_curand(tmp_path, seed):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import paper_1503_03769_b200 as phd
    n = 1_000_000
    c = _counters(n, seed & 0xFFFF)
    exe = str(tmp_path / "curand_kat")
    subprocess.check_call(["nvcc", "-O2", "-gencode", "arch=compute_100a,code=sm_100a", "-o", exe,
                           os.path.join(HERE, "pins", "curand_philox_kat.cu")])
    cin, cout = str(tmp_path / "c.bin"), str(tmp_path / "o.bin")
    c.tofile(cin)
    subprocess.check_call([exe, str(seed), cin, cout])
    ref = np.fromfile(cout, np.uint32).reshape(n, 4)
    dc = torch.from_numpy(c.view(np.int32)).cuda()
    do = torch.empty_like(dc)
    phd.philox_device(seed, dc, do)
    got = do.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, ref), int(np.sum(np.any(got != ref, axis=1)))
    # the host build of the same generator (pinned to ATen in test_abi / the oracle pins)
    key = [seed & 0xFFFFFFFF, seed >> 32]
    for i in np.random.default_rng(2).choice(n, 200, replace=False):
        assert phd.philox([int(v) for v in c[i]], key) == [int(v) for v in got[i]]
