"""Benchmark of the particle-PHD filter hot path (BASELINE.json metric:
"particle-measurement update pairs/sec and filter step ms at 1/2/4/8 B200").

Workload (N=1 and every N): config 5 "exchange stress" -- 2^24 particles
(16,711,680 survivors + 65,536 births), 4096 measurements per step, position
sensor; strong scaling over 1/2/4/8 GPUs.  One "step" = the
whole hot path (predict + births, two-pass update with its all-reduces, STPHD
extraction on rank 0, systematic resampling + exchange) via phd_step.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config cfg5] [--impl ours|reference]

Prints ONE JSON line on rank 0.  value = sum over timed steps of N*M pairs /
device time (CUDA events on the filter stream, barrier + synchronize on both
sides, max over ranks).  The particle state (335 MB) exceeds the 126 MB L2,
so no explicit flush is needed between steps.
"""
import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

# Per-pair algorithmic work of the two-pass update:
#   pass 1: 6 FP32 + 1 EX2 (position; +1 FP32 range-bearing)
#   pass 2: 6 FP32 + 1 EX2 for the weights (+1 range-bearing), plus 4 FP32 (+2 range-bearing
#           centring) for the STPHD state sums of the pairs whose label is in the estimated
#           index set I (fraction f = |I| / M); SURVEY.md §8(d) counted the state sums for
#           every pair (11 FP32), reported as "frac_survey_count".
FP32_PER_CLK_SM = 128.0   # measured: profiles/r01_pipes_microbench.jsonl (FFMA / FFMA2 lanes)
EX2_PER_CLK_SM = 16.0     # measured: MUFU.EX2
SM_MAX_MHZ = 1965.0
L2_BYTES = 126 * 2**20    # B200 L2


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="cfg5")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--mode", default="exact", choices=["exact", "dcp"],
                    help="exact: global C + exact resampling (north_star hot path); dcp: the paper's DCPFPHD groups")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--gate", type=int, default=0, choices=[0, 1, 2],
                    help="update algorithm of the main line: 0 dense (the pairs/s roofline line), 1/2 gated")
    ap.add_argument("--gate-floor", type=int, default=0,
                    help="gate_floor of the main line's gated update (0: exact gating; DESIGN.md §5)")
    ap.add_argument("--no-gated-leg", action="store_true",
                    help="skip the extra gated-update measurement reported under \"gated\"")
    ap.add_argument("--cpu-sample", type=int, default=65536, help="particles in the oracle's bounded sample")
    return ap.parse_args()


# Pass 1 evaluates 1/16 of its exp2 terms with an FMA-pipe polynomial (ex2_poly: 3 FADD
# + 5 FFMA per term) instead of MUFU.EX2: the joint FP32/EX2 bound counts both.
EMU_FRAC = 1.0 / 16.0
POLY_FP32 = 8.0


def emu_frac(meas):
    """share of pass-1 terms on the FMA polynomial (k_update.cu: every 4th particle's last
    slot pair of 4, i.e. 1/16; range-bearing every 8th: 1/32)"""
    return EMU_FRAC / 2 if meas == 1 else EMU_FRAC


def pass_ops(meas, which, f, hilo=False):
    """(FP32 ops, MUFU.EX2 ops) per pair.  hilo: also the seam-free hi/lo residual of the
    range-bearing sensor (+2 FP32 per pair per pass), implementation overhead rather than
    algorithmic work."""
    rb = 1 if meas == 1 else 0
    hl = 2 * rb if hilo else 0
    if which == "pass1":  # joint bound: the polynomial-offloaded terms move from EX2 to FP32
        return 6 + rb + hl + emu_frac(meas) * POLY_FP32, 1.0 - emu_frac(meas)
    if which == "pass2":
        return 6 + rb + hl + (4 + 2 * rb) * f, 1
    if which == "pass2_survey":
        return 11 + rb + hl, 1
    a, b = pass_ops(meas, "pass1", f, hilo), pass_ops(meas, "pass2", f, hilo)
    return a[0] + b[0], a[1] + b[1]


def roofline_pairs_per_s(meas, which, n_sm, mhz, f=1.0, hilo=False):
    fp, ex = pass_ops(meas, which, f, hilo)
    per_clk = min(FP32_PER_CLK_SM / fp, EX2_PER_CLK_SM / ex)
    return per_clk * n_sm * mhz * 1e6


def bound_of(meas, which, f, hilo=False):
    fp, ex = pass_ops(meas, which, f, hilo)
    return "alu:fp32" if fp / FP32_PER_CLK_SM >= ex / EX2_PER_CLK_SM else "alu:mufu.ex2"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    FIELDS = ["index", "clocks.sm", "clocks.max.sm", "power.draw", "clocks_event_reasons.active",
              "clocks_event_reasons.hw_slowdown", "clocks_event_reasons.hw_thermal_slowdown",
              "clocks_event_reasons.sw_thermal_slowdown", "clocks_event_reasons.sw_power_cap"]

    def __init__(self, devices):
        self.devices = devices
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "--query-gpu=" + ",".join(self.FIELDS), "--format=csv,noheader,nounits", "-lms", "200",
                 "-i", ",".join(str(d) for d in self.devices)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            # nvidia-smi's start-up (NVML init, driver locks) must not overlap the timed
            # region: it stalled the small configs' per-step CUDA calls (cfg 2 0.087 ->
            # 0.105 ms/step); wait for its first sample, then time
            t0 = time.time()
            while not self.rows and time.time() - t0 < 5.0 and self.proc.poll() is None:
                time.sleep(0.01)
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) == len(self.FIELDS):
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            for i, nm in enumerate(names):
                if r[5 + i].lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(self.rows)}


def scenario_for(name, steps):
    import scenario
    from dataclasses import replace
    cfg = scenario.get(name)
    if cfg.scenario.steps < steps:
        cfg = replace(cfg, scenario=replace(cfg.scenario, steps=steps))
    return cfg


def oracle_population_sample(cfg, truth, n):
    """The first n particles of the config's t = 0 population, from the oracle's own
    orc_init_population (cpu_baseline / reference arm only), each with the uniform share
    m0 / N_out of the mass (a timing sample: the mass box of cfg 5 would leave the
    lowest y-band with zero weight)."""
    import scenario
    import oracle
    ia = scenario.init_args(cfg, truth)
    n_out = scenario.initial_count(cfg, truth)[0]
    n = min(n, n_out)
    soa, w, _ = oracle.init_population(cfg.model, n_out, ia["box"], ia["v_max"], ia["total_mass"] * n / n_out,
                                       None, 0, n)
    import numpy as np
    return np.ascontiguousarray(soa.astype(np.float32)), np.ascontiguousarray(w.astype(np.float32)), n_out


def cpu_oracle_sample(cfg, Z, soa, w, n_sample, k=1):
    """The oracle, as it stands, on a bounded sample: one full serial step
    (predict, births, normalisers, update, extraction, resampling) of the
    first n_sample particles against the full measurement set Z_k."""
    import numpy as np
    import oracle
    m = cfg.model
    n = min(n_sample, soa.shape[1])
    sub = np.ascontiguousarray(soa[:, :n])
    ws = np.ascontiguousarray(w[:n])
    J = max(1, int(round(m.births_per_step * n / max(1, soa.shape[1]))))
    from dataclasses import replace
    ms = replace(m, births_per_step=J)
    z = Z[k - 1]
    t0 = time.perf_counter()
    r = oracle.step(ms, k, sub, ws, z, None, n, J)
    dt = time.perf_counter() - t0
    pairs = (n + J) * len(z)
    return {"pairs": pairs, "seconds": dt, "n": n + J, "M": len(z)}


def cpu_oracle_all_cores(cfg, Z, soa, w, n_sample, k=1):
    """Context, not the contract's cpu_baseline: the oracle's normaliser and update
    loops (the O(N M) part of a step) split over particles on every host core
    (oracle/phd_oracle_mt.c, fixed-order fp64 reduction), on a bounded sample."""
    import numpy as np
    import oracle
    m = cfg.model
    n = min(n_sample, soa.shape[1])
    nt = os.cpu_count() or 1
    sub = np.ascontiguousarray(soa[:, :n])
    ws = np.ascontiguousarray(w[:n]) + np.float32(1e-9)
    z = Z[k - 1]
    t0 = time.perf_counter()
    C = oracle.normalizers_mt(m, sub, ws, z, nt)
    oracle.update_mt(m, sub, ws, z, C, nt)
    dt = time.perf_counter() - t0
    pairs = n * len(z)
    return {"value": pairs / dt, "unit": "pairs/s", "cores": nt, "kind": "oracle (threaded timing variant)",
            "sample": "normalisers + weight/STPHD update of the first %d particles against all M=%d measurements "
                      "of Z_1, split over %d threads; %.1f s" % (n, len(z), nt, dt)}


def run_reference(args):
    import numpy as np
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    steps = args.warmup + args.steps
    cfg = scenario_for(args.config, steps)
    import scenario
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    n_s = 16384
    soa, w, _ = oracle_population_sample(cfg, truth, n_s)
    times, pairs = [], []
    for s in range(steps):
        r = cpu_oracle_sample(cfg, Z, soa, w, n_s, k=s + 1)
        if s >= args.warmup:
            times.append(r["seconds"])
            pairs.append(r["pairs"])
    T = sum(times)
    val = sum(pairs) / T
    sample = ("one full serial step (predict, births, normalisers, update, extraction, resampling) of the "
              "first %d particles (+ proportional births) against all M=%d measurements of Z_k, per step" %
              (n_s, len(Z[0])))
    out = {"impl": "reference", "metric": "particle-measurement update pairs/sec and filter step ms",
           "value": val, "unit": "pairs/s", "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * T / len(times), "higher_is_better": True, "scaling": "strong",
           "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "N": int(scenario.initial_count(cfg, truth)[0] + cfg.model.births_per_step),
                      "M": len(Z[0]), "sample_particles": n_s},
           "cpu_baseline": {"value": val, "unit": "pairs/s", "cores": 1, "kind": "oracle", "sample": sample},
           "e2e": {"value": val, "unit": "pairs/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)
    return 0


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        print("warning: --gpus %d but WORLD_SIZE %d" % (args.gpus, world), file=sys.stderr)
    if world > 1:  # NCCL's init log (transports, NVLS) stays visible on stderr for the scaling runs
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT,NVLS")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    import paper_1503_03769_b200 as phd
    import scenario
    phd.load(build_if_missing=(rank == 0 and world == 1))

    steps = args.warmup + args.steps
    cfg = scenario_for(args.config, 2 * steps + 1)
    from dataclasses import replace as _replace
    cfg = _replace(cfg, model=_replace(cfg.model, mode=1 if args.mode == "dcp" else 0, gate=args.gate,
                                           gate_floor=args.gate_floor))
    m = cfg.model
    truth = scenario.simulate_truth(cfg)
    Z = scenario.measurements(cfg, truth)
    ia = scenario.init_args(cfg, truth)   # t = 0 population recipe (phd_init_population)
    n0 = scenario.initial_count(cfg, truth)[0]
    J = m.births_per_step
    if args.mode == "dcp":   # every rank is one DCPFPHD group holding its block of the population
        lo, hi = phd.rank_block(n0, world, rank)
    else:
        lo, hi = phd.rank_block(n0 + J, world, rank)
    nid = None
    if world > 1:
        obj = [phd.nccl_unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nid = obj[0]
    # the filter's stream: a torch stream made current, so the CUDA events and the L2 flush
    # are ordered with the filter's kernels (handle 0, the legacy stream, would make the
    # library create a stream of its own)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    ws_bytes = phd.workspace_size(m, world)
    workspace = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)  # device memory from torch
    f = phd.Filter(m, rank=rank, world=world, nccl_id=nid, device=local, stream=stream.cuda_stream,
                   workspace=workspace)

    def reset():
        # the t = 0 population on the device (each DCP group: its block, full mass)
        f.init_population(**ia)

    # device-resident measurement sets (value) and pinned host copies (e2e)
    Zd = [torch.from_numpy(z).to(dev) for z in Z]
    Zh = [torch.from_numpy(z).pin_memory() for z in Z]

    def run_steps(kfirst, count, zs, timed):
        pairs = 0
        N_glob = n0 + J
        for i in range(count):
            k = kfirst + i
            z = zs[k - 1]
            M = int(z.shape[0])
            f.step_raw(k, z.data_ptr(), M)
            s = f._sum
            pairs += int(s.N) * M
        return pairs

    # Inputs smaller than L2 (configs 1-3): flush L2 before every timed step by
    # writing a buffer larger than it, outside that step's events; the step times
    # are summed.  Configs 4-5 stream more particle state than L2 holds.
    N_glob = n0 + J
    state_bytes = N_glob * 20
    flush = state_bytes < 2 * L2_BYTES
    flush_buf = torch.empty(2 * L2_BYTES, dtype=torch.uint8, device=dev) if flush else None

    def timed_steps(zs, kfirst, per_step=None):
        """K steps; returns (pairs, device ms).  barrier + synchronize on both sides."""
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)
        pairs, ms = 0, 0.0
        ev = []
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        if not flush:
            e0.record(stream)
        for i in range(args.steps):
            k = kfirst + i
            z = zs[k - 1]
            if flush:
                flush_buf.zero_()
                # wait for the flush: otherwise its tail overlaps the step (the library's
                # predict timer read ~50 us more) and hides the host's launch latency of the
                # step's first kernels, which a filter loop does pay (the GPU idles at the
                # step's start, after the previous step's estimates were read back)
                torch.cuda.synchronize(dev)
                a0, a1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a0.record(stream)
            f.step_raw(k, z.data_ptr(), int(z.shape[0]))
            if flush:
                a1.record(stream)
                ev.append((a0, a1))
            pairs += int(f._sum.N) * int(z.shape[0])
            if per_step is not None:
                per_step()
        if not flush:
            e1.record(stream)
        torch.cuda.synchronize(dev)
        if world > 1:
            dist.barrier()
        ms = sum(a.elapsed_time(b) for a, b in ev) if flush else e0.elapsed_time(e1)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return pairs, ms

    # ---- device-resident run (value): no per-kernel events in this timed region ----
    reset()
    run_steps(1, args.warmup, Zd, False)
    clocks = ClockSampler([local]) if rank == 0 else None
    if clocks:
        clocks.start()
    l0 = f.launch_count()
    g0_ = f.graph_stats()
    pairs, ms = timed_steps(Zd, args.warmup + 1)
    launches = f.launch_count() - l0
    g1_ = f.graph_stats()
    graph_info = {"captures_in_timed_steps": g1_[0] - g0_[0], "replays_in_timed_steps": g1_[1] - g0_[1],
                  "captures_total": g1_[0],
                  "note": "PHD_GRAPH=1: phd_step replays a CUDA graph of its kernel chain when one rank runs "
                          "the dense update (default: eager launches with programmatic dependent launch, "
                          "measured faster on B200); a new launch shape is captured once"}
    clk = clocks.stop() if clocks else None
    M = int(Z[0].shape[0])

    # ---- the same steps again with per-kernel CUDA events (kernel_ms, roofline) ----
    pass_ms = {"pass1": [], "pass2": [], "update": [], "predict": [], "resample": [], "exchange": []}

    def collect():
        t = f.timing()
        for key in pass_ms:
            pass_ms[key].append(t[key])

    reset()
    run_steps(1, args.warmup, Zd, False)
    f.set_timing(True)
    timed_steps(Zd, args.warmup + 1, collect)
    f.set_timing(False)

    # ---- e2e: host measurement buffers, copies inside the timed region ----
    reset()
    run_steps(1, args.warmup, Zh, False)
    pairs_e, ms_e = timed_steps(Zh, args.warmup + 1)

    # ---- near-tie counts (north_star: resampled indices bit-exact except thresholds within
    # 1e-9 of a cumulative-sum boundary, "with that count reported"; S8 label sets) ----
    # one more step through the separate calls, after the timed regions: the weights the
    # kernels resampled are read back and the thresholds near a boundary counted on the host
    near = None
    if args.mode == "exact":
        from paper_1503_03769_b200.diag import resample_near_ties, label_threshold_near_ties
        kx = args.warmup + args.steps + 1
        f.predict(kx)
        f.update(Z[kx - 1])
        _, wn_loc, _ = f.get_particles()
        _, sx = f.extract()
        lab = label_threshold_near_ties(f.accumulators(int(Z[kx - 1].shape[0]))[:, 0], int(sx["LT"])) \
            if rank == 0 else None
        f.resample_exchange(kx)
        anc_loc, first = f.ancestors()
        meta = f.resample_meta()
        O_r = float(sum(meta["W_r"][:rank]))
        ties = int(np.sum(resample_near_ties(wn_loc, meta["U"], meta["N_out"], W=meta["W"], O=O_r,
                                             j_lo=first, j_hi=first + len(anc_loc))))
        if world > 1:
            t = torch.tensor([ties], device=dev, dtype=torch.int64)
            dist.all_reduce(t)
            ties = int(t.item())
        near = {"step": kx, "resample_thresholds_within_1e-9": ties, "N_out": int(meta["N_out"]),
                "label_threshold_near_ties": lab, "LT": int(sx["LT"]),
                "basis": "thresholds t_j = (j+U)W/N_out within 1e-9 (unnormalised mass) of a cumulative sum of "
                         "the resampled fp32 weights (where the GPU's fp64 scan order may pick the neighbour); "
                         "labels whose dW is within 1e-5 relative of the LT-th (S8). Ancestor mismatches vs the "
                         "oracle are checked element-wise in tests/test_gpu_parity.py::test_full_size_sampled"}

    # ---- gated update (NEXT-2): same workload, same steps, gate = 1 ----
    # exact gating (every skipped term underflows to 0), then with gate_floor F = log2(kappa) - 60
    # (skipped terms < 2^F: every C(z) within N 2^F <= 2^-36 kappa of the exact one at N <= 2^24)
    gated = gated_floor = None
    if not args.no_gated_leg and args.gate == 0:
        def gated_leg(mg, note):
            nonlocal f, workspace, nid
            f.close()
            workspace = None  # released before the next filter's workspace
            if world > 1:  # an NCCL unique id bootstraps one communicator: a fresh one for this filter
                obj = [phd.nccl_unique_id() if rank == 0 else None]
                dist.broadcast_object_list(obj, src=0)
                nid = obj[0]
            workspace = torch.empty(phd.workspace_size(mg, world), dtype=torch.uint8, device=dev)
            f = phd.Filter(mg, rank=rank, world=world, nccl_id=nid, device=local, stream=stream.cuda_stream,
                           workspace=workspace)
            reset()
            run_steps(1, args.warmup, Zd, False)
            g_st = []
            pairs_g, ms_g = timed_steps(Zd, args.warmup + 1, lambda: g_st.append(f.gate_stats()))
            g_ms = {"pass1": [], "pass2": [], "update": []}

            def collect_g():
                t = f.timing()
                for key in g_ms:
                    g_ms[key].append(t[key])

            reset()
            run_steps(1, args.warmup, Zd, False)
            f.set_timing(True)
            timed_steps(Zd, args.warmup + 1, collect_g)
            f.set_timing(False)
            ev = sum(s_["pairs"] for s_ in g_st)
            return {"ms_per_step": ms_g / args.steps,
                    "effective_pairs_per_s": pairs_g / (ms_g * 1e-3),
                    "evaluated_pairs_per_step": ev / max(1, len(g_st)),
                    "evaluated_fraction": ev / max(1, pairs_g // max(1, world)),
                    "steps_gated": sum(s_["used"] for s_ in g_st),
                    "kernel_ms": {k_: statistics.mean(v_) for k_, v_ in g_ms.items()},
                    "pass_roofline": None,
                    "note": note}

        gated = gated_leg(_replace(m, gate=1),
                          "gate = 1: only (tile, measurement) pairs whose largest exponent is >= -130 are "
                          "evaluated (every skipped term is exactly 0 in fp32 ftz); effective = N*M / step time, "
                          "not a pairs/s roofline claim")
        V = (m.region[1] - m.region[0]) * (m.region[3] - m.region[2])
        kap = m.clutter_rate / V if V > 0 else 0.0
        if kap > 0:
            F = max(-126, min(-20, int(math.floor(math.log2(kap))) - 60))
            gated_floor = gated_leg(_replace(m, gate=1, gate_floor=F),
                                    "gate = 1, gate_floor = %d = floor(log2 kappa) - 60: pairs whose largest "
                                    "term is below 2^%d are skipped too, so every C(z) is within N 2^%d "
                                    "(<= 2^-36 kappa) of the exact gating (parity: test_gate_floor_parity)"
                                    % (F, F, F))
            gated_floor["gate_floor"] = F
            gated_floor["C_abs_bound"] = float(n0 + J) * 2.0 ** F

    # per-rank stage times (max / mean over ranks): passes, resampling, exchange incl. its
    # barrier, and the share of particles each rank updated (load balance)
    per_rank = None
    if world > 1:
        mine = {k_: statistics.mean(v_) for k_, v_ in pass_ms.items()}
        mine["particles"] = float(hi - lo)
        if gated is not None:  # the gated update's evaluated pairs on this rank (its candidate balance)
            mine["gated_evaluated_pairs"] = float(gated["evaluated_pairs_per_step"])
        allr = [None] * world
        dist.all_gather_object(allr, mine)
        per_rank = {k_: {"max": max(r_[k_] for r_ in allr), "mean": statistics.mean(r_[k_] for r_ in allr),
                         "per_rank": [r_[k_] for r_ in allr]} for k_ in mine}
        per_rank["exchange_path"] = f.exchange_path()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return 0

    value = pairs / (ms * 1e-3)
    value_e = pairs_e / (ms_e * 1e-3)
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    for gl in (gated, gated_floor):
        if gl is None or gl["evaluated_pairs_per_step"] <= 0:
            continue
        # evaluated pairs per gated pass against the same EX2-bound pair roofline as the dense passes
        evp = gl["evaluated_pairs_per_step"]
        r1 = evp / (gl["kernel_ms"]["pass1"] * 1e-3)
        r2 = evp / (gl["kernel_ms"]["pass2"] * 1e-3)
        pk = roofline_pairs_per_s(m.meas, "pass1", n_sm, SM_MAX_MHZ)
        gl["pass_roofline"] = {"unit": "Gpair/s (evaluated)", "peak": pk / 1e9,
                               "pass1": r1 / 1e9, "pass1_frac": r1 / pk,
                               "pass2": r2 / 1e9, "pass2_frac_of_ex2_bound": r2 / pk,
                               "basis": "1 MUFU.EX2 per evaluated pair per pass, 16/clk/SM x %d SMs x %.0f MHz; "
                                        "pass 2 also carries the state sums of the index set"
                                        % (n_sm, SM_MAX_MHZ)}
    mhz = (clk or {}).get("sm_mhz") or SM_MAX_MHZ
    p2 = statistics.mean(pass_ms["pass2"])
    p1 = statistics.mean(pass_ms["pass1"])
    local_pairs = (hi - lo) * M
    n_sel = min(int(f._sum.LT), M)
    frac_sel = (n_sel / M) if (M and m.stphd_all == 0) else 1.0
    ach2 = local_pairs / (p2 * 1e-3)
    peak2 = roofline_pairs_per_s(m.meas, "pass2", n_sm, SM_MAX_MHZ, frac_sel)
    peak2_survey = roofline_pairs_per_s(m.meas, "pass2_survey", n_sm, SM_MAX_MHZ)
    ach_upd = local_pairs / ((p1 + p2) * 1e-3)
    peak_upd = roofline_pairs_per_s(m.meas, "update", n_sm, SM_MAX_MHZ, frac_sel)
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(cfg.name, {}).get("k_pass2")
        except Exception:
            traffic = None
    # HBM-bound steps (north_star: predict / resample achieved GB/s against the B200 peak):
    # algorithmic bytes per launch / mean event time; peak = MEASURED_PEAKS.json hbm_gbs
    hbm_peak = 6460.5
    try:
        hbm_peak = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
        peak_src = "MEASURED_PEAKS.json hbm_gbs (torch copy, read+write bytes)"
    except Exception:
        peak_src = "fallback 6460.5 GB/s"
    n_loc = hi - lo
    n_surv_loc = max(0, min(hi, n0) - min(lo, n0))
    rb_bytes = 32 if m.meas == 1 else 0
    b_pred = n_surv_loc * (40 + rb_bytes) + (n_loc - n_surv_loc) * (20 + rb_bytes)
    b_res = n_loc * 20 + n0 // world * 24
    t_pred = statistics.mean(pass_ms["predict"])
    t_res = statistics.mean(pass_ms["resample"])
    hbm = {"peak_gbs": hbm_peak, "peak_basis": peak_src,
           "predict": {"bytes": b_pred, "ms": t_pred, "gbs": b_pred / (t_pred * 1e6), "frac": b_pred / (t_pred * 1e6) / hbm_peak,
                       "basis": "survivor 40 B (state + w read and written), birth 20 B written%s" %
                                (", + 32 B range-bearing representation" if rb_bytes else "")},
           "resample": {"bytes": b_res, "ms": t_res, "gbs": b_res / (t_res * 1e6), "frac": b_res / (t_res * 1e6) / hbm_peak,
                        "basis": "per particle w + state read (20 B); per offspring state + w written (20 B) and the "
                                 "ancestor index (4 B); k_scan_chunks + k_resample_gather (both kernels)"}}
    cpu = None
    cpu_all = None
    if not args.no_cpu_baseline and world == 1:  # the contract's CPU baseline: rank 0 at N = 1 only
        soa, w, _ = oracle_population_sample(cfg, truth, args.cpu_sample * 4)
        r = cpu_oracle_sample(cfg, Z, soa, w, args.cpu_sample, k=1)
        full_pairs = N_glob * M
        cpu = {"value": r["pairs"] / r["seconds"], "unit": "pairs/s", "cores": 1, "kind": "oracle",
               "sample": "one full serial fp64 step (predict, births, normalisers, update, extraction, resampling) "
                         "of the first %d particles of the t=0 population (+%d proportional births) against all "
                         "M=%d measurements of Z_1; %.1f s" % (args.cpu_sample, r["n"] - args.cpu_sample, r["M"],
                                                               r["seconds"]),
               "extrapolated_full_step_s": full_pairs / (r["pairs"] / r["seconds"]),
               "extrapolated_note": "EXTRAPOLATED, not measured: N*M = %d pairs of one full step at the sample's "
                                    "pairs/s (the step is O(N M); its O(N) parts are < 1%% at this M)" % full_pairs}
        cpu_all = cpu_oracle_all_cores(cfg, Z, soa, w, args.cpu_sample * 4)
        cpu_all["extrapolated_full_step_s"] = full_pairs / cpu_all["value"]
    out = {
        "metric": "particle-measurement update pairs/sec and filter step ms",
        "value": value, "unit": "pairs/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic",
        "config": {"workload": cfg.name, "N": N_glob, "M": M, "survivors": n0, "births": J,
                   "meas_model": "position" if m.meas == 0 else "range_bearing", "parallelism": "dp%d" % world,
                   "mode": args.mode,
                   "l2": ("L2 flushed before every timed step (%d MB write; particle state %.1f MB < 126 MB L2); "
                          "step times summed" % (2 * L2_BYTES >> 20, state_bytes / 2**20)) if flush else
                         ("inputs larger than L2 (particle state %d MB > 126 MB)" % (state_bytes >> 20))},
        "update_pairs_per_s": local_pairs * world / ((statistics.mean(pass_ms["update"])) * 1e-3),
        "kernel_ms": {k: statistics.mean(v) for k, v in pass_ms.items()},
        "roofline": {"bound": bound_of(m.meas, "pass2", frac_sel), "kernel": "k_pass<pass 2> (weights + STPHD sums)",
                     "achieved": ach2 / 1e9, "peak": peak2 / 1e9, "unit": "Gpair/s", "frac": ach2 / peak2,
                     "traffic": traffic,
                     "peak_basis": "min(128 FP32 lanes / %.2f, 16 EX2 / 1) per SM-clk x %d SMs x %.0f MHz (max clock); "
                                   "%.2f FP32 = %s, f = |I|/M = %.3f (state sums for the estimated index set); "
                                   "pipe rates measured (profiles/r01_pipes_microbench.jsonl)"
                                   % (pass_ops(m.meas, "pass2", frac_sel)[0], n_sm, SM_MAX_MHZ,
                                      pass_ops(m.meas, "pass2", frac_sel)[0],
                                      "7 + 6 f (range-bearing: + anisotropy multiply, + centring on the "
                                      "Cartesian image; the hi/lo residual is not counted)"
                                      if m.meas == 1 else "6 + 4 f", frac_sel),
                     "frac_at_observed_clock": ach2 / roofline_pairs_per_s(m.meas, "pass2", n_sm, mhz, frac_sel),
                     "frac_with_hilo_ops": (ach2 / roofline_pairs_per_s(m.meas, "pass2", n_sm, SM_MAX_MHZ, frac_sel, True))
                     if m.meas == 1 else None,
                     "frac_survey_count": ach2 / peak2_survey},
        "update_roofline": {"achieved": ach_upd / 1e9, "peak": peak_upd / 1e9, "unit": "Gpair/s",
                            "frac": ach_upd / peak_upd, "bound": bound_of(m.meas, "update", frac_sel),
                            "basis": "joint FP32/EX2 bound of both passes: (%s) FP32 + (2 - 1/16) EX2 per pair "
                                     "(pass 1 evaluates 1/16 of its terms with an 8-FP32 polynomial), f = %.3f"
                                     % ("14.5 + 6 f" if m.meas == 1 else "12.5 + 4 f", frac_sel),
                            "pass1": {"achieved": local_pairs / (p1 * 1e-3) / 1e9,
                                      "peak": roofline_pairs_per_s(m.meas, "pass1", n_sm, SM_MAX_MHZ) / 1e9,
                                      "frac": local_pairs / (p1 * 1e-3) / roofline_pairs_per_s(m.meas, "pass1", n_sm,
                                                                                                SM_MAX_MHZ),
                                      "bound": bound_of(m.meas, "pass1", frac_sel)},
                            "frac_with_hilo_ops": (ach_upd / roofline_pairs_per_s(m.meas, "update", n_sm, SM_MAX_MHZ,
                                                                                  frac_sel, True))
                            if m.meas == 1 else None,
                            "hilo_note": "range-bearing: the seam-free hi/lo residual adds 2 FP32 per pair per pass "
                                         "(implementation overhead, not counted in 'frac'; 'frac_with_hilo_ops' counts it)"
                            if m.meas == 1 else None,
                            "frac_vs_survey_17fp32_2ex2": ach_upd / (min(FP32_PER_CLK_SM / 17.0, EX2_PER_CLK_SM / 2.0)
                                                                     * n_sm * SM_MAX_MHZ * 1e6)},
        "cpu_baseline": cpu,
        "cpu_baseline_all_cores": cpu_all,
        "e2e": {"value": value_e, "unit": "pairs/s", "h2d_bytes_per_step": M * 8,
                "d2h_bytes_per_step": int(f._sum.n_est) * 24 + 8 * (2 * world + 10)},
        "gpu_launches": int(launches),
        "paper_context": {"hardware": "a Dell computer using MATLAB (PAPER.md:494); no CPU model, cores or "
                                      "precision stated",
                          "workload": "BOT range-bearing scenario, 2000 particles, K = 4 groups, 50 scans "
                                      "(PAPER.md:444-448)",
                          "table1_dcpphd_speedup_vs_phd": {"r=0": 2.04, "r=10": 2.66, "r=20": 2.97},
                          "note": "Table 1 (PAPER.md:497-513), context only: not this metric or workload"},
        "hbm_kernels": hbm,
        "gated": gated,
        "gated_floor": gated_floor,
        "per_rank": per_rank,
        "graph_steps": graph_info,
        "near_ties": near,
        "clocks": clk,
    }
    print(json.dumps(out), flush=True)
    f.close()
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
