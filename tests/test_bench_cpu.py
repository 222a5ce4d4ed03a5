"""bench.py's reference arm runs on the host alone: its JSON line keeps the driver contract."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line(ref):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference"
    assert line["metric"].startswith("expEuler steps/s")
    assert line["unit"] == "steps/s" and line["higher_is_better"] is True
    assert line["steps"] == 2 and line["warmup"] == 1 and line["n_gpus"] == 1
    assert len(line["step_seconds"]) == 2 and abs(line["ms_per_step"] / 1e3 - sum(line["step_seconds"]) / 2) < 1e-9
    assert "full 32x32x32 grid" in line["cpu_baseline"]["sample"]
    assert line["value"] > 0
    cb = line["cpu_baseline"]
    assert cb["kind"] == "reference" and cb["cores"] >= 1 and cb["value"] == line["value"]
    assert line["e2e"] == {"value": line["value"], "unit": "steps/s", "h2d_bytes_per_step": 0,
                           "d2h_bytes_per_step": 0}
    assert line["config"]["workload"].startswith("C1")


def test_reference_arm_non_zero_ranks_exit_quietly(ref):
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "1", "--warmup", "0"], capture_output=True, text=True, timeout=600, cwd=ROOT,
                         env=env)
    assert out.returncode == 0, out.stderr[-2000:]
    assert out.stdout.strip() == ""


def test_algorithmic_byte_models():
    """The roofline's byte models (pure functions of the step log): the fused two-term sweeps
    and the 2-D kernel's four-term rounds."""
    sys.path.insert(0, ROOT)
    import bench
    # stages of 5, 4 and 3 terms: 3 + 2 + 2 sweeps; the stage after the 4-term one starts from an
    # implicit f = F + T
    b, sweeps, implicit = bench.taylor_bytes_per_voxel([5, 4, 3])
    assert (sweeps, implicit) == (7, 1)
    assert b == bench.BYTES_FIRST_ZERO + bench.BYTES_PER_SWEEP * 6 + bench.BYTES_IMPLICIT
    b2, rounds, _ = bench.flat2d_bytes_per_voxel([12, 11, 4, 1])
    assert rounds == 3 + 3 + 1 + 1
    assert b2 == rounds * (8 * 5 + 8 * 1600 / 1024)
    assert "fits the 126 MB L2" in bench.l2_note(128 ** 3) and "no flush needed" in bench.l2_note(256 ** 3)


def test_default_step_counts():
    """Without --steps the headline config and the reference arm time 10 steps; the small
    configs their own run length."""
    sys.path.insert(0, ROOT)
    import bench
    from paper_2402_02273_b200 import workloads as W
    for cfg, impl, want in (("C4", "ours", 10), ("C2", "ours", 200), ("C5", "ours", 50), ("C2", "reference", 10)):
        w = W.get(cfg)
        steps = 10 if (impl == "reference" or w.n >= 256 ** 3) else w.steps
        assert steps == want
