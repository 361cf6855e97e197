"""Multi-rank host logic on CPU (gloo, world_size 2 and 3; -m "not gpu").

Each rank holds its contiguous block of a global weight array, all-gathers the
per-rank masses, takes its resampling bounds and its exchange plan from the C
library's host helpers (phd_resample_bounds, phd_plan_exchange), resamples
rank-locally with the same fp64 offset/pinning arithmetic the CUDA kernels use
(DESIGN.md §4), and exchanges offspring with gloo send/recv.  The gathered
result must equal the serial oracle's systematic resampling (exact except
thresholds within rounding of a cumulative-sum boundary), and every rank must
end with exactly its block of the next step's array.
"""
import math
import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _n_of(B, scale, U, lo, hi):
    t = B * scale - U
    c = math.ceil(t)
    return min(max(c, lo), hi)


def rank_local_resample(w_local, g0, O_r, scale, U, lo, hi, blk=1024):
    """numpy mirror of k_scan_blocks + k_resample_mark + max-scan: offspring ancestors."""
    n = len(w_local)
    nprod = hi - lo
    marks = np.full(nprod, -1, dtype=np.int64)
    nb = (n + blk - 1) // blk
    blk_sums = [math.fsum(w_local[b * blk:(b + 1) * blk]) for b in range(nb)]
    off = np.concatenate([[0.0], np.cumsum(blk_sums)])
    for b in range(nb):
        Eb = O_r + off[b]
        nEb = lo if b == 0 else _n_of(Eb, scale, U, lo, hi)
        nEb1 = hi if b == nb - 1 else _n_of(O_r + off[b + 1], scale, U, lo, hi)
        seg = w_local[b * blk:(b + 1) * blk]
        L = np.cumsum(seg)
        run = nEb
        prev = nEb
        for k in range(len(seg)):
            i = b * blk + k
            h = nEb1 if (i == n - 1 or k == blk - 1) else _n_of(Eb + L[k], scale, U, nEb, nEb1)
            run = max(run, h)
            if run > prev:
                marks[prev - lo] = g0 + i
            prev = run
    return np.maximum.accumulate(marks) if nprod else marks


def _worker(rank, world, port, seed, n, n_out, J, q):
    import torch.distributed as dist
    import torch
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1503_03769_b200 as phd
        import oracle
        rng = np.random.default_rng(seed)
        w = rng.uniform(0, 1, n) * (rng.uniform(size=n) < 0.5)
        w[: n // 2] *= 0.01  # imbalance: most mass on the upper ranks
        lo_b, hi_b = phd.rank_block(n, world, rank)
        wl = w[lo_b:hi_b]
        Wr = torch.tensor([math.fsum(wl)], dtype=torch.float64)
        allW = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allW, Wr)
        W_r = np.array([t.item() for t in allW])
        U = oracle.resample_U(seed, 5)
        bounds, W = phd.resample_bounds(W_r, n_out, U)
        O_r = 0.0
        for r in range(rank):
            O_r += W_r[r]
        anc = rank_local_resample(wl, lo_b, O_r, n_out / W, U, int(bounds[rank]), int(bounds[rank + 1]))
        # exchange: offspring -> owners of the next array [0, n_out) within blocks of n_out + J
        sc, so, rc, ro = phd.plan_exchange(world, rank, bounds, n_out, J)
        nlo, nhi = phd.rank_block(n_out + J, world, rank)
        mine = np.full(max(0, min(nhi, n_out) - min(nlo, n_out)), -7, dtype=np.int64)
        reqs = []
        for qd in range(world):
            if qd == rank:
                if sc[qd]:
                    mine[ro[qd]:ro[qd] + rc[qd]] = anc[so[qd]:so[qd] + sc[qd]]
                continue
            if sc[qd]:
                reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(anc[so[qd]:so[qd] + sc[qd]])), qd))
        for qd in range(world):
            if qd != rank and rc[qd]:
                buf = torch.zeros(int(rc[qd]), dtype=torch.int64)
                dist.recv(buf, qd)
                mine[ro[qd]:ro[qd] + rc[qd]] = buf.numpy()
        for r_ in reqs:
            r_.wait()
        parts = [None] * world
        dist.all_gather_object(parts, (nlo, mine.tolist(), int(bounds[rank + 1] - bounds[rank])))
        if rank == 0:
            q.put((w.tolist(), U, parts, bounds.tolist()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,n_out,J", [(2, 5000, 4200, 300), (3, 7001, 6000, 101)])
def test_sharded_resampling_equals_serial(orc, world, n, n_out, J):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, 17, n, n_out, J, q)) for r in range(world)]
    for p in procs:
        p.start()
    w, U, parts, bounds = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    w = np.array(w)
    # every rank holds exactly its block of the next step's survivors, in global order
    glob = []
    for r, (nlo, mine, nprod) in enumerate(sorted(parts, key=lambda t: t[0])):
        assert min(nlo, n_out) == len(glob)
        assert -7 not in mine
        glob.extend(mine)
    assert len(glob) == n_out and sum(p[2] for p in parts) == n_out
    ser, _ = orc.resample(w, U, n_out)
    glob = np.array(glob)
    mism = np.nonzero(glob != ser)[0]
    B = np.cumsum(w)
    t = (np.arange(n_out) + U) * B[-1] / n_out
    for j in mism:
        assert np.min(np.abs(B - t[j])) <= 1e-9 * B[-1], (j, glob[j], ser[j])
    assert len(mism) <= 2
