"""The bench.py JSON-line contract (task statement, "Measurement"): the keys the
driver reads, their types and the relations between them.  The reference arm
(the oracle on the host cores) runs here on the CPU; our arm on the GPU."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config"}


def run_bench(args, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                       timeout=timeout, env=e, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    return [json.loads(ln) for ln in lines]


def test_reference_arm_line():
    """--impl reference: the oracle as it stands on a bounded sample, one JSON line
    with the base keys, impl, cpu_baseline (kind oracle, cores, sample) and an e2e
    with zero copy bytes, value = cpu_baseline.value = e2e.value."""
    (d,) = run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0"])
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["unit"] == "MLUPS" and d["higher_is_better"] is True and d["value"] > 0
    assert d["steps"] == 1 and d["warmup"] == 0 and d["n_gpus"] == 1
    cb = d["cpu_baseline"]
    assert cb["kind"] == "oracle" and cb["cores"] >= 1 and cb["sample"] and cb["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "MLUPS", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}


def test_reference_arm_non_zero_rank_prints_nothing():
    """Under torchrun only rank 0 runs the reference arm; the other ranks exit 0
    without work or output."""
    assert run_bench(["--impl", "reference", "--steps", "1", "--warmup", "0", "--gpus", "2"],
                     env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"}) == []


@pytest.mark.gpu
def test_our_arm_line():
    """Our arm at the bench workload, few steps: base keys; roofline frac =
    achieved / peak with the measured peak; warm-up honoured; kernel launches
    counted; e2e through host buffers with the state bytes each way; clocks
    sampled; cpu_baseline from the oracle."""
    (d,) = run_bench(["--steps", "4", "--warmup", "3"])
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["steps"] == 4 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["dtype"] == "f64"
    assert d["config"]["lattice"] == [512, 512, 64]
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert 0.3 < r["frac"] < 1.0
    with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
        assert r["peak"] == json.load(fh)["hbm_gbs"]
    assert abs(d["value"] - 512 * 512 * 64 / (d["ms_per_step"] * 1e-3) / 1e6) < 1e-6 * d["value"]
    assert d["gpu_launches"] >= d["steps"]
    e = d["e2e"]
    state = 2 * 19 * 512 * 512 * 64 * 8
    assert e["h2d_bytes_per_step"] == state and e["d2h_bytes_per_step"] == state and 0 < e["value"] < d["value"]
    assert d["clocks"]["sm_mhz"] > 0 and "reasons" in d["clocks"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
