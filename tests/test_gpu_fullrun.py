"""North_star's full-run parity gate on BASELINE.json's configurations, against the compiled,
unmodified reference (`gliosim::run`, /root/reference/proj/src/integrator.cpp:91-138, built
into oracle/_ref by oracle/Makefile) and the pinned C restatement (per-step decisions).

| config | what runs                                    | steps            |
|--------|----------------------------------------------|------------------|
| C1     | 32^3 shell phantom (single-cluster path)     | 100 (full run)   |
| C2     | 256^2 mid-plane slice                        | 200 (full run)   |
| C3     | 128^3 from a 29-slice stack, two seeds       | 100 (full run)   |
| C4     | 256^3 perturbed phantom                      | 10 (trajectory)  |
| C4x4   | 256^3 at 4x rho                              | 5 (trajectory)   |
| C5     | 4 ensemble members (min/mid/max rho, random) | 50 (full run)    |

Every test asserts (tests/fullrun.py): material map memcmp-equal to the reference's
resample; per step, (s, m) and terms per stage equal the oracle's on the GPU's own input and
u within relative L2 1e-10; the production gs_run loop bitwise equal to the stepwise one;
final u within relative L2 1e-8 of the reference's run() and total mass within 1e-8 at
every node.  The whole 100-step C4 comparison is tools/fullrun_record.py (minutes of
reference time on the host cores) -> profiles/r02_c4_trajectory_parity.json.

Set FULLRUN_RECORD_DIR to keep each test's JSON record.
"""
import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import fullrun as FR  # noqa: E402

pytestmark = pytest.mark.gpu


def _save(rec):
    out = os.environ.get("FULLRUN_RECORD_DIR")
    if out:
        os.makedirs(out, exist_ok=True)
        with open(os.path.join(out, f"fullrun_{rec['config']}.json"), "w") as f:
            json.dump(rec, f, indent=1, default=str)


def _case(name):
    import bench
    from paper_2402_02273_b200 import workloads as W
    w = W.get(name)
    data, dims, labels = bench.build_case(w)
    op = bench.make_operator(w, data, dims)
    return w, data, dims, op


def _material_gate(ref, w, data, dims, op):
    """The device material map (K1) memcmp-equal to the reference's resample + classify
    (imaging.cpp:118-141) of the same bytes -- at C3 the 128x128x29 -> 128^3 z-upsampling."""
    want = ref.resample(data, dims[0], dims[1], dims[2], (w.nx, w.ny, w.nz))
    got = op.labels()
    assert got.tobytes() == want.tobytes(), int(np.sum(got != want))
    return got


@pytest.mark.parametrize("name,steps", [("C1", 100), ("C2", 200), ("C3", 100), ("C4", 10), ("C4x4", 5)])
def test_full_run_matches_reference(name, steps, port, ref):
    import bench
    from paper_2402_02273_b200 import workloads as W
    w, data, dims, op = _case(name)
    try:
        labels = _material_gate(ref, w, data, dims, op)
        u0 = bench.initial_state(w, op, labels)
        center = W.seed_points(w, labels)[0]
        rec = FR.full_run_parity(name, op, labels, u0, steps, w.rho, w.tau, W.TOL, center, port, ref)
        rec["material_map_equal"] = True
        rec["path"] = ("single-cluster" if op.uses_cluster() else
                       "resident tiles (2-D)" if op.uses_flat2d() else "multi-kernel")
        _save(rec)
        FR.assert_record(rec)
    finally:
        op.close()


def test_c5_members_full_run_match_reference(port, ref):
    """C5: four members of the real ensemble -- lowest, middle and highest rho plus one seeded
    random member -- advanced all 50 steps by the batched ensemble (gs_run_ensemble), each
    against the reference's run() of that member; per-step decisions and the 1e-10 bar in
    one-step mode on the batched path's own states."""
    from paper_2402_02273_b200 import ensemble as E
    from paper_2402_02273_b200 import gliosim as G
    from paper_2402_02273_b200 import phantom
    from paper_2402_02273_b200 import workloads as W
    w = W.get("C5")
    steps = w.steps
    rhos = [W.member_rho(w, mb) for mb in range(w.members)]
    pick = [int(np.argmin(rhos)), w.members // 2, int(np.argmax(rhos))]
    rnd = int(phantom.uniform01(w.seed, 77, 1)[0] * w.members)
    while rnd in pick:
        rnd = (rnd + 1) % w.members
    pick.append(rnd)
    runner = E.EnsembleRunner(w, pick)
    try:
        ops_o = []
        for mb, op in zip(pick, runner.ops):
            data, wd, ht, sl = W.intensity(w, mb)
            labels = _material_gate(ref, w, data, (wd, ht, sl), op)
            ops_o.append(port.stencil((w.nx, w.ny, w.nz), w.h, port.diffusion_from_labels(labels)))

        def states():
            runner.reset()
            prev = [np.array(u, copy=True) for u in runner.u0]
            for k in range(steps):
                _, inf = G.run_ensemble(runner.ops, 1, runner.rhos, w.tau, W.TOL, metrics=False, infos=True)
                for i, op in enumerate(runner.ops):
                    nxt = op.get_state()
                    yield (i, k), inf[i][0], prev[i], nxt, ops_o[i], runner.rhos[i]
                    prev[i] = nxt

        rec = dict(config="C5", members=pick, member_rhos=runner.rhos, steps=steps)
        rows = FR.check_one_step_sequence(port, None, states(), None, w.tau, W.TOL, record=rec)
        stepwise = [op.get_state() for op in runner.ops]
        rec["per_step_max_rel_l2"] = max(r["rel_l2"] for r in rows)
        rec["per_step_decisions_equal"] = all(r["gpu"] == r["oracle"] for r in rows)
        rec["per_step_bitwise"] = all(r["bitwise"] for r in rows)
        runner.reset()
        met, inf = G.run_ensemble(runner.ops, steps, runner.rhos, w.tau, W.TOL, np.zeros((len(pick), 3)),
                                  np.array(runner.centers), 0.1, metrics=True, infos=True)
        finals = []
        for i, (mb, op) in enumerate(zip(pick, runner.ops)):
            u_gpu = op.get_state()
            assert FR.bitwise(u_gpu, stepwise[i]), f"member {mb}: batched 50-step run != stepwise run"
            prod = [FR._info_tuple(x) for x in inf[i]]
            assert prod == [tuple(r["gpu"]) for r in rows if r["key"][0] == i]
            d = port.diffusion_from_labels(op.labels())
            u_ref, m_ref, _ = ref.run(op.grid.shape, w.h, d, runner.u0[i], steps, runner.rhos[i], W.T0,
                                      W.T0 + steps * w.tau, W.TOL, runner.centers[i], 0.1, workers=FR.host_cores())
            m_gpu = np.array([[x.total_mass, x.max_density, x.min_density, x.radius] for x in met[i]])
            finals.append(dict(member=mb, rho=runner.rhos[i], final_rel_l2_vs_reference=FR.rel_l2(u_gpu, u_ref),
                               final_bitwise_vs_reference=FR.bitwise(u_gpu, u_ref),
                               nan_voxels=int(np.isnan(u_gpu).sum()),
                               metrics_mass_max_rel_diff=FR.compare_metrics(m_gpu[:, 0], m_ref[:, 0]),
                               terms_per_step=[int(sum(t[2])) for t in prod]))
        rec["members_final"] = finals
        _save(rec)
        assert rec["per_step_decisions_equal"], [r["key"] for r in rec["per_step"] if not r["decisions_equal"]][:10]
        assert rec["per_step_max_rel_l2"] <= FR.PER_STEP_TOL
        assert rec["per_step_bitwise"]
        for f in finals:
            assert f["final_rel_l2_vs_reference"] <= FR.FULL_RUN_TOL, f
            assert f["final_bitwise_vs_reference"], f
            assert f["metrics_mass_max_rel_diff"] <= 1e-8, f
    finally:
        runner.close()
