"""bench.py keeps the driver's JSON contract: our arm (GPU) and the reference
arm (the CPU oracle port, runs here)."""
import json
import os
import subprocess
import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
BASE_KEYS = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
             "vs_baseline", "dtype", "data", "config", "e2e"}


def _run(*args, timeout=600):
    env = dict(os.environ, RANK="0", WORLD_SIZE="1")
    r = subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], cwd=ROOT, env=env, capture_output=True,
                       text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    return json.loads(lines[0])


def _check_e2e(d):
    e = d["e2e"]
    assert {"value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"} <= set(e)
    assert e["unit"] == d["unit"] and e["value"] > 0


def test_reference_arm_json():
    d = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0", timeout=300)
    assert BASE_KEYS <= set(d) and d["impl"] == "reference"
    assert d["metric"] == "masked tokens/sec scored (logprob+GRPO loss)" and d["higher_is_better"] is True
    assert d["value"] > 0 and d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cores"] >= 1
    _check_e2e(d)
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the same config dict our arm prints for this workload (it names the workload; "run" says how)
    sys.path.insert(0, str(ROOT))
    import bench
    from paper_2603_18815_b200 import synth
    c = synth.CONFIGS["c1"]
    g = bench.global_workload(c, 1, "weak")
    sh = synth.make_shard(g, seed=2603 + c["index"])
    assert d["config"] == bench.workload_config(c, "c1", g, 1, "weak", len(sh.groups), sh.n_active)
    assert d["cpu_baseline"]["timing"] == "wall clock" and d["cpu_baseline"]["cpu_model"]


@pytest.mark.gpu
def test_bench_json_contract():
    d = _run("--steps", "3", "--warmup", "3", "--no-cpu-baseline", "--no-backward")
    assert BASE_KEYS <= set(d) and "impl" not in d
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["scaling"] == "weak"
    assert d["data"].startswith("synthetic") and d["dtype"] == "bf16" and "workload" in d["config"]
    _check_e2e(d)
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-9
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])
    assert "cpu_baseline" in d
