"""The reference's own acceptance program (/root/reference/proj/tests/acceptance.cpp, compiled
unmodified by `make -C oracle accept`) run twice on the B200 box:

* oracle/_ref/acceptance_ref    -- linked against the whole reference (CPU);
* oracle/_ref/acceptance_dropin -- the same program with the reference's exponential
  integrator (expact.o, integrator.o) replaced at link time by tests/cpp/acceptance_shim.cpp,
  i.e. every expmv / phi1v / step / run of the criteria (and of pipeline.cpp's
  run_to_directory and wave_speed_experiment) runs on the GPU drop-in.

Every criterion the reference passes must pass on the drop-in: c1 exponential-action kernels
(50 random operators), c2 100 steps == one action, c3 conservation and stability, c4
traveling-wave speed, c5 first-order convergence over 25-200 steps, c6 benchmark report, c7
bytewise determinism, c8 the 29-slice imaging pipeline.
"""
import os
import re
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_ref")
GPU_BIN = os.path.join(ROOT, "oracle", "_ref", "acceptance_dropin")
LINE = re.compile(r"^\[(PASS|FAIL)\] criterion (\d+): (.*)$")


def _run(exe):
    if not os.path.exists(exe):
        pytest.skip(f"{os.path.basename(exe)} not built (make -C oracle accept needs the reference sources)")
    out = subprocess.run([exe], capture_output=True, text=True, timeout=1500, cwd=ROOT)
    res = {}
    for ln in out.stdout.splitlines():
        m = LINE.match(ln.strip())
        if m:
            res[int(m.group(2))] = (m.group(1) == "PASS", m.group(3))
    return out, res


def test_acceptance_criteria_on_the_dropin():
    ref_out, ref = _run(REF_BIN)
    gpu_out, gpu = _run(GPU_BIN)
    print(ref_out.stdout)
    print(gpu_out.stdout)
    assert ref and set(gpu) == set(ref), (sorted(ref), sorted(gpu), gpu_out.stderr[-2000:])
    for cid, (ok, detail) in sorted(ref.items()):
        if ok:
            assert gpu[cid][0], f"criterion {cid} passes on the reference but not on the drop-in: {gpu[cid][1]}"
    assert gpu_out.returncode == 0 or not all(ok for ok, _ in ref.values())
