"""C-ABI library: loads, exports every symbol include/phd.h declares, and its
host-only helpers are right (-m "not gpu"; no compute call needs a GPU)."""
import ctypes
import math
import os
import re

import numpy as np
import pytest

import paper_1503_03769_b200 as phd
from paper_1503_03769_b200 import binding

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "phd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(phd_[a-z0-9_]+)\s*\(", src)))


def test_library_loads_and_exports_header_symbols():
    L = phd.load()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(binding.EXPORTS)
    assert L.phd_abi_version() == binding.ABI_VERSION == 3
    assert L.phd_status_str(2) == b"call out of order"


def test_params_struct_layout_matches_header(tmp_path):
    """The ctypes mirror of phd_params / phd_summary / phd_estimate has the C layout
    (sizeof and every field offset, compiled from include/phd.h with gcc)."""
    import subprocess
    structs = {"phd_params": binding.Params, "phd_summary": binding.Summary, "phd_estimate": binding.Estimate}
    lines = ['#include <stdio.h>', '#include <stddef.h>', '#include "phd.h"', "int main(void) {"]
    for cname, py in structs.items():
        lines.append('printf("%s sizeof %%zu\\n", sizeof(%s));' % (cname, cname))
        for fname, _ in py._fields_:
            lines.append('printf("%s %s %%zu\\n", offsetof(%s, %s));' % (cname, fname, cname, fname))
    lines.append("return 0; }")
    src = tmp_path / "layout.c"
    src.write_text("\n".join(lines))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)])
    out = subprocess.run([str(exe)], stdout=subprocess.PIPE, check=True).stdout.decode().split("\n")
    got = {tuple(l.split()[:2]): int(l.split()[2]) for l in out if l.strip()}
    for cname, py in structs.items():
        assert got[(cname, "sizeof")] == ctypes.sizeof(py), cname
        for fname, _ in py._fields_:
            assert got[(cname, fname)] == getattr(py, fname).offset, (cname, fname)


def test_host_philox_matches_oracle(orc):
    rng = np.random.default_rng(2)
    for _ in range(500):
        ctr = [int(v) for v in rng.integers(0, 2**32, 4)]
        key = [int(v) for v in rng.integers(0, 2**32, 2)]
        assert phd.philox(ctr, key) == orc.philox(ctr, key)


def test_rank_block_partition():
    for n in [0, 1, 7, 1000, 2**24, 2**24 + 3]:
        for world in [1, 2, 3, 4, 8]:
            prev = 0
            for r in range(world):
                lo, hi = phd.rank_block(n, world, r)
                assert lo == prev and lo == (n * r) // world and hi == (n * (r + 1)) // world
                prev = hi
            assert prev == n


def test_resample_bounds_tile_and_match_serial(orc):
    """n(O_r) bounds: rank r produces exactly the offspring whose thresholds fall in its mass."""
    rng = np.random.default_rng(9)
    for trial in range(20):
        world = int(rng.integers(1, 9))
        n = int(rng.integers(world, 400))
        w = rng.uniform(0, 1, n) * (rng.uniform(size=n) < 0.6)
        w[int(rng.integers(0, n))] += 0.5
        n_out = int(rng.integers(1, 600))
        U = orc.resample_U(trial, 2)
        W_r = [math.fsum(w[(n * r) // world:(n * (r + 1)) // world]) for r in range(world)]
        b, W = phd.resample_bounds(W_r, n_out, U)
        assert b[0] == 0 and b[-1] == n_out and np.all(np.diff(b) >= 0)
        # serial oracle ancestors: the offspring of rank r's particles are exactly [b[r], b[r+1])
        # except at thresholds within rounding of a rank boundary (counted, must be rare)
        anc, _ = orc.resample(w, U, n_out)
        owner = np.searchsorted([(n * (r + 1)) // world for r in range(world)], anc, side="right")
        mism = 0
        for r in range(world):
            mism += int(np.sum(owner[b[r]:b[r + 1]] != r))
        assert mism <= 2


def test_plan_exchange_conserves():
    rng = np.random.default_rng(4)
    for _ in range(50):
        world = int(rng.integers(1, 9))
        n_out = int(rng.integers(0, 5000))
        J = int(rng.integers(0, 300))
        cuts = np.sort(rng.integers(0, n_out + 1, world - 1))
        bounds = np.concatenate([[0], cuts, [n_out]]).astype(np.int64)
        sends = np.zeros((world, world), dtype=np.int64)
        recvs = np.zeros((world, world), dtype=np.int64)
        for r in range(world):
            sc, so, rc, ro = phd.plan_exchange(world, r, bounds, n_out, J)
            sends[r] = sc
            recvs[r] = rc
            assert sc.sum() == bounds[r + 1] - bounds[r]
            lo, hi = phd.rank_block(n_out + J, world, r)
            assert rc.sum() == max(0, min(hi, n_out) - min(lo, n_out))
            # receive segments are disjoint and ordered by source rank (order-preserving)
            segs = [(ro[q], ro[q] + rc[q]) for q in range(world) if rc[q] > 0]
            for (a0, a1), (b0, b1) in zip(segs, segs[1:]):
                assert a1 == b0
        assert np.array_equal(sends, recvs.T)


def test_create_without_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    import scenario
    m = scenario.get("cfg1").model
    with pytest.raises(phd.PhdError) as e:
        phd.Filter(m)
    assert e.value.status in (6, 8)  # PHD_ECUDA / PHD_ENODEV


def test_invalid_params_rejected():
    import scenario
    from dataclasses import replace
    m = scenario.get("cfg1").model
    for bad in [replace(m, sigma_z=(0.0, 10.0)), replace(m, p_d=1.5), replace(m, births_per_step=0),
                replace(m, max_meas=0), replace(m, T=0.0)]:
        with pytest.raises(phd.PhdError) as e:
            phd.workspace_size(bad)
        assert e.value.status == 1
