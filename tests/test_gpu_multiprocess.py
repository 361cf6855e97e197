"""The multi-process data plane on one GPU (-m gpu): world = 2 and 3 processes, each with
its own filter context on cuda:0, collectives through a test-only host transport
(torch.distributed gloo; NCCL refuses several ranks on one device).  What runs is the
product path of one process per GPU: the CUDA-IPC peer window
(cudaIpcGetMemHandle / cudaIpcOpenMemHandle across processes), the fused resampling
gather storing offspring into the other processes' next-step buffers, the
double-buffer flips, the rank-local exact resampling.  The result must equal the
1-process run (fp64 summation order only; counted near-ties in the ancestors), itself
pinned to the oracle by test_gpu_parity.py (the exchange of Step 6)."""
import os
import socket
from dataclasses import replace

import numpy as np
import pytest

import scenario
from scenario.configs import COUNT_FIXED

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _cfg():
    cfg = scenario.get("cfg3")
    m = replace(cfg.model, fixed_count=60000, births_per_step=4096, capacity=64096, count_mode=COUNT_FIXED,
                max_meas=4096)
    s = replace(cfg.scenario, n_targets=40, steps=4, init_mass_box=(0.0, 1000.0, 0.0, 1000.0),
                start_box=(0.0, 1000.0, 0.0, 1000.0))
    return replace(cfg, model=m, scenario=s)


def _run(rank, world, port, steps, out, xch):
    """One rank (world > 1: a spawned process with a gloo group); writes its results to out."""
    import sys
    sys.path.insert(0, ROOT)
    import torch
    import paper_1503_03769_b200 as phd
    if xch == "nccl":  # the send/recv exchange through the host transport
        os.environ["PHD_EXCHANGE"] = "nccl"
    t = None
    if world > 1:
        import torch.distributed as dist
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)

        def allreduce(vals):
            g = [None] * world
            dist.all_gather_object(g, list(vals))
            acc = np.array(g[0], np.float64)
            for r in range(1, world):  # rank order
                acc = acc + np.array(g[r], np.float64)
            return acc.tolist()

        def allgather(b):
            g = [None] * world
            dist.all_gather_object(g, b)
            return g

        t = phd.host_transport(allreduce, allgather)
    torch.cuda.set_device(0)
    cfg = _cfg()
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    f = phd.Filter(cfg.model, rank=rank, world=world, device=0, transport=t)
    f.init_population(**scenario.init_args(cfg, truth))
    res = {}
    for k in range(1, steps + 1):
        s = f.step(k, Z[k - 1]).as_dict()
        a, first = f.ancestors()
        p, w, g0 = f.get_particles()
        res["W%d" % k] = s["W"]
        res["LT%d" % k] = s["LT"]
        res["anc%d" % k] = a
        res["first%d" % k] = first
        res["pop%d" % k] = p
        res["w%d" % k] = w
        res["g0%d" % k] = g0
        if rank == 0:
            res["lab%d" % k] = f.estimates()["labels"]
    res["xpath"] = f.exchange_path()
    f.close()
    np.savez(out, **res)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world,xch", [(2, "p2p"), (3, "p2p"), (2, "nccl")])
def test_multiprocess_ipc_exchange_equals_one_process(tmp_path, world, xch):
    import torch
    import torch.multiprocessing as mp
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    steps = 3
    ref = str(tmp_path / "ref.npz")
    ctx = mp.get_context("spawn")
    p = ctx.Process(target=_run, args=(0, 1, 0, steps, ref, xch))
    p.start()
    p.join(600)
    assert p.exitcode == 0
    port = _free_port()
    outs = [str(tmp_path / ("r%d.npz" % r)) for r in range(world)]
    procs = [ctx.Process(target=_run, args=(r, world, port, steps, outs[r], xch)) for r in range(world)]
    for q in procs:
        q.start()
    for q in procs:
        q.join(600)
    assert all(q.exitcode == 0 for q in procs), [q.exitcode for q in procs]
    R = np.load(ref)
    G = [np.load(o) for o in outs]
    assert int(G[0]["xpath"]) == (2 if xch == "p2p" else 1)  # the IPC peer window was set up across processes
    n_out = _cfg().model.fixed_count
    identical = True
    for k in range(1, steps + 1):
        anc = np.concatenate([g["anc%d" % k] for g in sorted(G, key=lambda g: int(g["first%d" % k]))])
        pop = np.concatenate([g["pop%d" % k] for g in sorted(G, key=lambda g: int(g["g0%d" % k]))], axis=1)
        w = np.concatenate([g["w%d" % k] for g in sorted(G, key=lambda g: int(g["g0%d" % k]))])
        assert len(anc) == n_out and pop.shape == R["pop%d" % k].shape
        # every rank holds its block of the next step's array (the exchange moved the offspring)
        for r, g in enumerate(G):
            lo = (n_out + 4096) * r // world
            assert int(g["g0%d" % k]) == lo
        if identical:
            assert abs(float(G[0]["W%d" % k]) - float(R["W%d" % k])) <= 1e-6 * max(1.0, float(R["W%d" % k]))
            assert int(G[0]["LT%d" % k]) == int(R["LT%d" % k])
            mism = np.mean(anc != R["anc%d" % k])
            assert mism <= 4e-4, mism
            same = np.all(pop == R["pop%d" % k], axis=0)
            assert np.mean(same) >= 1 - 4e-4
            # the offspring states are the ancestors' states, stored by the other processes
            assert np.allclose(w, R["w%d" % k], rtol=1e-6)
            identical = bool(np.all(anc == R["anc%d" % k]))
