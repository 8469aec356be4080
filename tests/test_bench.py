"""Host-side checks of bench.py (no GPU): the workload table, the byte accounting behind
roofline.frac, the reference arm's JSON line, and that our arm fails loudly without a GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from oracle import ft_oracle as fo  # noqa: E402


def test_workloads_are_the_baseline_configs():
    # BASELINE.json configs 1-5 (sigma, d, l, storage, sweeps per step)
    want = {"config1": (2, 2, 8, "f64", 500), "config2": (3, 3, 4, "f64", 300),
            "config3": (4, 2, 8, "f32", 100), "config4": (2, 2, 17, "f32", 50),
            "config5": (2, 2, 18, "f32", 30)}
    for name, (s, d, ell, dt, sw) in want.items():
        w = bench.WORKLOADS[name]
        assert (w["sigma"], w["d"], w["ell"], w["dtype"], w["sweeps"]) == (s, d, ell, dt, sw)
    for w in bench.WORKLOADS.values():  # every form is one the oracle accepts for (sigma, d)
        fo.resolve_form(w["sigma"], w["d"], w["form"])


def test_algorithmic_bytes():
    w4 = bench.WORKLOADS["config4"]
    stored = 3229614080  # quarter table of l = 17, K = 7 (tests/test_quarter.py)
    assert bench.algorithmic_bytes_for_kernel(w4, stored, "bin2q") == 2 * stored * 4
    # every logical window of the half table (2^33 entries) + every stored entry written
    assert bench.requested_bytes_per_sweep(w4, stored, "bin2q") == (1 << 33) * 4 + stored * 4
    w3 = bench.WORKLOADS["config3"]
    half = 1 << 31  # complement-folded 4^16 / 2
    # read v_{n-1} and the row means of v_{n-2}, write v_n and its row means
    assert bench.algorithmic_bytes_for_kernel(w3, half, "q4") == 2 * half * 4 + 2 * (half // 16) * 8
    assert bench.algorithmic_bytes_for_kernel(bench.WORKLOADS["config3ta"], half, "q4") == \
        bench.algorithmic_bytes_for_kernel(w3, half, "q4")


def test_workload_name_is_shared_by_both_arms():
    class A:
        workload = "config3"
    name = bench.workload_name(A, bench.WORKLOADS["config3"])
    assert name.startswith("config3: sigma=4, d=2, l=8, ks form, f32 storage, 100 sweeps")


def _run(args, timeout=300):
    env = dict(os.environ, CUDA_VISIBLE_DEVICES="")
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                          capture_output=True, text=True, timeout=timeout, env=env)


def test_reference_arm_prints_one_json_line():
    r = _run(["--impl", "reference", "--workload", "config1", "--steps", "1", "--warmup", "3"])
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    res = json.loads(lines[0])
    assert res["impl"] == "reference" and res["unit"] == "state-updates/s" and res["value"] > 0
    assert res["cpu_baseline"]["kind"] == "oracle" and res["cpu_baseline"]["cores"] >= 1
    assert res["e2e"]["h2d_bytes_per_step"] == 0 and res["e2e"]["value"] == res["value"]
    assert res["config"]["workload"].startswith("config1:")


@pytest.mark.skipif(os.environ.get("LCSB_TEST_HAS_GPU") == "1", reason="CPU-only check")
def test_our_arm_fails_loudly_without_a_gpu():
    r = _run(["--workload", "config1", "--steps", "1", "--warmup", "3", "--no-cpu-baseline"])
    assert r.returncode != 0
    assert not [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
