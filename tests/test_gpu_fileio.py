"""GPU side of SURVEY.md 8(f) #2 and #4: run_to_directory with the asynchronous snapshot
sink, device matter_fractions, and PGM-stack ingest straight into the device material map.

Parity: snapshot files hold exactly the states the GPU run produced (checked bitwise
against states captured through the synchronous sink, and byte-for-byte against
correctly rounded '%.17g' formatting); the run itself is checked against the C oracle
within the per-run tolerance of 1e-8 (relative L2); labels and fractions are exact.
"""
import os

import numpy as np
import pytest

from paper_2402_02273_b200 import gliosim as G, phantom

pytestmark = pytest.mark.gpu


def tiny_config():
    """test_pipeline.cpp:22-35."""
    return G.SimConfig(nx=8, ny=8, nz=1, h=200.0 / 7.0, t0=0.0, t_end=200.0, num_steps=4, snapshot_every=2,
                       seed_center=(100.0, 100.0, 0.0), seed_amplitude=0.5, seed_width=0.002)


def vtk_body(path, n):
    with open(path) as f:
        lines = f.read().split("\n")
    return lines[10:10 + n]


def test_run_to_directory_writes_snapshots_and_metrics(tmp_path, port):
    """test_pipeline.cpp:51-76."""
    cfg = tiny_config()
    g = cfg.grid()
    d = G.uniform_diffusion(g, cfg.d_white)
    out = tmp_path / "outdir"
    seen = []
    res = G.run_to_directory(cfg, d, None, out, 1, on_step=seen.append)
    assert len(seen) == cfg.num_steps
    for k in (0, 2, 4):
        assert (out / f"snapshot_{k:04d}.vtk").exists()
    for k in (1, 3):
        assert not (out / f"snapshot_{k:04d}.vtk").exists()
    assert (out / "metrics.csv").exists()
    last = G.read_vtk(out / "snapshot_0004.vtk")
    assert np.array_equal(last.values.view(np.uint64), res.u.view(np.uint64))  # text round trip is exact
    assert len(res.metrics) == 5
    rows = (out / "metrics.csv").read_text().splitlines()
    assert rows[0] == "step,time_days,total_mass,max_density,radius_mm"
    for m, row in zip(res.metrics, rows[1:]):
        assert row == ",".join([str(m.step)] + ["%.17g" % x for x in (m.time, m.total_mass, m.max_density,
                                                                        m.radius)])
    # the run against the oracle (per-run bar)
    op = port.stencil(g.shape, g.h, d.d)
    u0 = port.seed_initial(g.shape, g.h, cfg.seed_amplitude, cfg.seed_width, cfg.seed_center, d_mask=d.d)
    want, _, _ = port.run(op, u0, cfg.num_steps, cfg.rho, cfg.tau(), cfg.exp_tol, cfg.seed_center)
    assert np.linalg.norm(res.u - want) <= 1e-8 * np.linalg.norm(want)


def test_run_to_directory_embeds_material_array(tmp_path):
    """test_pipeline.cpp:78-91."""
    cfg = tiny_config()
    g = cfg.grid()
    d = G.uniform_diffusion(g, cfg.d_white)
    mv = G.uniform_labels(g, 1)
    G.run_to_directory(cfg, d, mv, tmp_path / "o")
    text = (tmp_path / "o" / "snapshot_0000.vtk").read_text()
    assert "SCALARS material int 1" in text


def test_async_snapshots_hold_exactly_the_run_states(tmp_path):
    """64^3 phantom, a snapshot every step so several are in flight at once: every file is
    the state of its step (captured independently through the synchronous sink) to the bit,
    formatted exactly as printf('%.17g')."""
    n = 64
    h = 200.0 / (n - 1)
    inten = phantom.shell_phantom(n, n, n, seed=8).ravel()
    grid = G.Grid(n, n, n, h)
    i, j, k = n // 2, n // 2, n // 2
    cfg = G.SimConfig(nx=n, ny=n, nz=n, h=h, num_steps=6, snapshot_every=1, seed_center=(i * h, j * h, k * h),
                      seed_amplitude=1.0, seed_width=1.0 / (2.0 * (3.0 * h) ** 2))
    states = {}
    with G.StencilOperator.from_intensity(grid, inten, n, n, n) as op:
        labels = op.labels()
        u0 = G.seed_initial(op, cfg)
        G.run(cfg, op, u0, snapshot=lambda s, t, u: states.__setitem__(s, u.copy()))
        res = G.run_to_directory(cfg, op, labels, tmp_path / "o")
    assert res.timings.io_seconds > 0
    for s in range(cfg.num_steps + 1):
        p = tmp_path / "o" / f"snapshot_{s:04d}.vtk"
        f = G.read_vtk(p)
        assert np.array_equal(f.values.view(np.uint64), states[s].view(np.uint64)), s
        if s in (0, cfg.num_steps):
            body = vtk_body(p, 2 * n ** 3 + 2)
            assert body[:n ** 3] == ["%.17g" % x for x in states[s]]
            assert body[n ** 3:n ** 3 + 2] == ["SCALARS material int 1", "LOOKUP_TABLE default"]
            assert body[n ** 3 + 2:] == [str(int(x)) for x in labels]


def test_snapshot_to_unwritable_path_fails_at_the_call(tmp_path):
    with G.StencilOperator.from_labels(G.Grid(8, 8, 8, 1.0), np.ones(512, np.uint8)) as op:
        op.set_state(np.zeros(512))
        with pytest.raises(G.DataError, match="cannot open .* for writing"):
            op.snapshot_vtk(tmp_path / "missing" / "s.vtk")
        op.snapshot_vtk(tmp_path / "ok.vtk")
        op.flush_snapshots()
    assert G.read_vtk(tmp_path / "ok.vtk").values.sum() == 0.0


def test_matter_fractions_on_device(port):
    n = 48
    inten = phantom.shell_phantom(n, n, n, seed=2).ravel()
    with G.StencilOperator.from_intensity(G.Grid(n, n, n, 1.0), inten, n, n, n) as op:
        w, g = G.matter_fractions(op)
        lab = op.labels()
    cnt = np.bincount(lab, minlength=4)
    tissue = int(cnt[1] + cnt[2])
    assert (w, g) == (float(cnt[1]) / tissue, float(cnt[2]) / tissue)  # imaging.cpp:163 arithmetic
    with pytest.raises(G.DataError, match="no tissue voxels"):
        G.matter_fractions(G.MaterialVolume(G.Grid(4, 4, 4, 1.0), np.zeros(64, np.uint8)))


def test_pgm_stack_ingest_into_device_material_map(tmp_path, port):
    """Full-resolution ingest: a 532x565x29 PGM stack read by the native
    loader, resampled and classified on the GPU; labels bit-identical to the oracle."""
    w, hgt, slices = 532, 565, 29
    stack = phantom.slice_stack(w, hgt, slices, 120, seed=6)
    paths = []
    for s in range(slices):
        p = tmp_path / f"slice_{s:03d}.pgm"
        p.write_bytes(f"P5\n# slice {s}\n{w} {hgt}\n255\n".encode() + stack[s].tobytes())
        paths.append(p)
    st = G.load_stack(paths)
    assert (st.width, st.height, st.num_slices) == (w, hgt, slices)
    assert np.array_equal(st.intensities, stack.ravel())
    for shape in ((64, 64, 64), (100, 90, 29)):
        grid = G.Grid(*shape, 1.0)
        with G.stencil_from_stack(st, grid) as op:
            got = op.labels()
            fr = G.matter_fractions(op)
        want = port.resample(st.intensities, w, hgt, slices, shape)
        assert np.array_equal(got, want), shape
        cnt = np.bincount(want, minlength=4)
        assert fr == (float(cnt[1]) / (cnt[1] + cnt[2]), float(cnt[2]) / (cnt[1] + cnt[2]))
    # raw-volume route: the same intensities through load_raw_volume
    raw = tmp_path / "vol.raw"
    raw.write_bytes(f"{w} {hgt} {slices}\n".encode() + stack.tobytes())
    st2 = G.load_raw_volume(raw)
    assert np.array_equal(st2.intensities, st.intensities)


def test_gpu_formatter_matches_host_formatter_on_every_value_class(tmp_path):
    """The device %.17g (gs_vtkfmt.cu) against the host writer (exact fmt17 + glibc for the
    special values) on random bit patterns, subnormals, huge and tiny magnitudes, integers,
    signed zeros, infinities and NaNs of both signs: byte-identical files."""
    n = 64 * 64 * 16
    rng = np.random.default_rng(12)
    bits = rng.integers(0, 2 ** 63, n, dtype=np.int64).view(np.uint64) ^ (rng.integers(0, 2, n).astype(np.uint64) << np.uint64(63))
    v = bits.view(np.float64).copy()
    k = n // 8
    v[:k] = rng.uniform(0, 1, k)
    v[k:2 * k] = rng.uniform(-1, 1, k) * 10.0 ** rng.integers(-320, 300, k)
    v[2 * k:2 * k + 1000] = rng.integers(-10 ** 9, 10 ** 9, 1000)
    special = [0.0, -0.0, np.inf, -np.inf, np.nan, -np.nan, 5e-324, -5e-324, 2.2250738585072014e-308,
               1.7976931348623157e308, 1e16, 1e17, 9.999999999999999e-5, 1e-4, 0.1, 1.0 / 3]
    v[3 * k:3 * k + len(special)] = special
    labels = rng.integers(0, 4, n).astype(np.uint8)
    grid = G.Grid(64, 64, 16, 0.5, (1.0, -2.0, 0.25))
    with G.StencilOperator.from_labels(grid, labels) as op:
        op.set_state(v)
        op.snapshot_vtk(tmp_path / "gpu.vtk", labels)
        op.flush_snapshots()
    G.write_vtk(G.ScalarField(grid, v), tmp_path / "host.vtk", labels)
    assert (tmp_path / "gpu.vtk").read_bytes() == (tmp_path / "host.vtk").read_bytes()
