"""bench.py on CPU: the reference arm (the oracle) prints one JSON line with the
contract keys, and the roofline helpers are consistent (-m "not gpu")."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "3", "--config", "cfg1"], stdout=subprocess.PIPE, stderr=subprocess.PIPE,
                       text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.strip().splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"


def test_roofline_helpers():
    sys.path.insert(0, ROOT)
    import bench
    # state sums for every pair (f = 1.25 -> 12.5 + 5 = 17.5 FP32 incl. the 1/16 polynomial
    # offload of pass 1): FP32-bound at 128/17.5 pairs/clk/SM
    assert abs(bench.roofline_pairs_per_s(0, "update", 148, 1965, 1.25) - 128 / 17.5 * 148 * 1965e6) < 1
    # state sums for a quarter of the pairs: EX2-bound, 2 - 1/16 EX2 per pair (joint bound)
    assert abs(bench.roofline_pairs_per_s(0, "update", 148, 1965, 0.25) - 16 / 1.9375 * 148 * 1965e6) < 1
    assert abs(bench.roofline_pairs_per_s(0, "pass1", 148, 1965) - 16 / (15 / 16) * 148 * 1965e6) < 1
    assert bench.bound_of(0, "pass2", 0.25) == "alu:mufu.ex2" and bench.bound_of(0, "pass2", 1.0) == "alu:fp32"
    # range-bearing: the hi/lo residual ops are counted only on request
    assert bench.pass_ops(1, "pass2", 0.0, hilo=True)[0] == bench.pass_ops(1, "pass2", 0.0)[0] + 2
