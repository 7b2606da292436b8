"""bench.py's reference arm runs on the host alone (it times the CPU oracle port), so its JSON
line can be checked here against the driver's contract."""

from __future__ import annotations

import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def test_reference_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", "--steps", "1",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for key in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
                "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert key in d, key
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "TFLOP/s"
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


import pytest  # noqa: E402


@pytest.mark.gpu
def test_main_arm_prints_one_contract_line():
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--steps", "3", "--warmup", "3", "--no-extra",
                          "--no-cpu"], cwd=ROOT, capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches",
                "speedup_vs_padded", "memory_saved_pct"):
        assert key in d, key
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["gpu_launches"] == 127 * 3
    r = d["roofline"]
    assert r["bound"] in ("tensor", "hbm") and 0 < r["frac"] <= 1 and r["peak"] > 0
    e = d["e2e"]
    assert e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0 and 0 < e["value"] < d["value"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(d["clocks"])


def test_gpus_n_spawns_n_ranks_and_prints_one_line():
    """`bench.py --gpus 2` without a torchrun environment spawns 2 ranks itself (the driver's
    `--gpus N` contract); the plumbing (rendezvous on 127.0.0.1, barrier-bracketed timing, max
    over ranks, one line from rank 0) is exercised on CPU over gloo with --dry-run."""
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "2", "--dry-run", "--steps", "2",
                          "--warmup", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["dry_run"] is True and d["steps"] == 2
    assert d["config"]["parallelism"].startswith("ep2")


def test_gpus_mismatch_with_world_size_fails_loudly():
    import os

    env = dict(os.environ, WORLD_SIZE="1", RANK="0", LOCAL_RANK="0")
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--gpus", "4", "--dry-run"], cwd=ROOT,
                         capture_output=True, text=True, timeout=120, env=env)
    assert out.returncode != 0 and "WORLD_SIZE" in out.stderr


def test_reference_arm_config_is_the_main_arm_config():
    sys.path.insert(0, str(ROOT))
    import bench

    ref = bench.headline_config(1, False)
    assert ref["workload"].startswith("residual sweep") and ref["N"] == 4096 and ref["K"] == 7168
    # both arms draw the headline operands from the same seed: identical bytes
    a = bench.headline_operands(bench.HEADLINE_SEED, 64, n=256, k=256)
    b = bench.headline_operands(bench.HEADLINE_SEED, 64, n=256, k=256)
    for x, y in zip(a, b):
        assert x.tobytes() == y.tobytes()
    assert not any(((c & 0x7F) == 0x7F).any() for c in (a[0], a[2]))  # no NaN code
