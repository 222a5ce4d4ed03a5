"""GPU parity: the CUDA path (through the C-ABI) against the oracle and the reference's
golden vectors.

Bars (BASELINE.json north_star): material map and (s, m) sequence exact; u within a
relative L2 error of 1e-10 per step and 1e-8 after a full run.  Beyond that, with the
device's tree-reduced ||b||_1 and bordered column sum fed to the oracle, every Taylor
term is reproduced BIT-FOR-BIT (those two sums are the only order-
dependent reductions on the path).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

STEP_TOL = 1e-10   # relative L2 per step (north_star)
RUN_TOL = 1e-8     # relative L2 after the full run (north_star)


@pytest.fixture(scope="module")
def G():
    from paper_2402_02273_b200 import gliosim
    return gliosim


def rel_l2(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def case(runs_kat, name):
    p = name + "."
    shape = tuple(int(v) for v in runs_kat[p + "shape"])
    h, rho, tau, tol, width, cx, cy, cz = (float(v) for v in runs_kat[p + "params"])
    return dict(shape=shape, h=h, rho=rho, tau=tau, tol=tol, width=width, center=(cx, cy, cz),
                labels=runs_kat[p + "labels"], states=runs_kat[p + "states"], metrics=runs_kat[p + "metrics"],
                log=runs_kat[p + "log"])


RUN_NAMES = ["r16", "r2d", "rtau", "rs9", "r4rho", "runmasked", "rflat"]


# ---- material map (K1) ----------------------------------------------------------------

def test_material_map_stack29(G, material_kat):
    stack = material_kat["stack29"]
    for shape, key in [((24, 20, 40), "stack29.labels"), ((17, 31, 9), "stack29.labels_xy")]:
        labels = G.resample(stack, 24, 20, 29, G.Grid(*shape, h=1.0))
        assert np.array_equal(labels, material_kat[key]), key


def test_material_map_nearest_kats(G, material_kat):
    for src in range(1, 8):
        px = np.array([0 if s % 2 == 0 else 100 for s in range(src)], dtype=np.uint8)
        for n in range(1, 8):
            got = G.resample(px, src, 1, 1, G.Grid(n, 1, 1, 1.0))
            assert np.array_equal(got, material_kat[f"nn.{src}.{n}"]), (src, n)


def test_classify_all_intensities(G, material_kat):
    stack = np.arange(256, dtype=np.uint8)
    labels = G.resample(stack, 256, 1, 1, G.Grid(256, 1, 1, 1.0))
    assert np.array_equal(labels, material_kat["classify"])


def test_diffusion_from_labels_matches_reference(G, material_kat):
    labels = material_kat["stack29.labels"]
    with G.StencilOperator.from_labels(G.Grid(24, 20, 40, 1.0), labels) as op:
        assert np.array_equal(op.diffusion(), material_kat["stack29.d"])
        assert np.array_equal(op.labels(), labels)


# ---- operator: apply and exact 1-norm ----------------------------------------------------

def test_stencil_apply_and_norm_bitwise(G, kat):
    for i in range(int(kat["stencil.count"][0])):
        p = f"stencil.{i}"
        shape = tuple(int(v) for v in kat[p + ".shape"])
        with G.assemble_diffusion(G.Grid(*shape, h=float(kat[p + ".h"][0])), kat[p + ".d"]) as op:
            assert np.array_equal(op.apply(kat[p + ".x"]), kat[p + ".Ax"]), p
            assert op.one_norm() == kat[p + ".A.norm1"][0], p


def test_fp64_field_mode_matches_oracle(G, port):
    """> 256 distinct D values: the operator runs on the fp64 D field instead of the palette."""
    rng = np.random.default_rng(3)
    shape = (19, 13, 11)
    n = np.prod(shape)
    d = np.where(rng.random(n) < 0.2, 0.0, rng.uniform(0.01, 0.2, n))
    x = rng.uniform(-1, 1, n)
    op_o = port.stencil(shape, 1.3, d)
    with G.assemble_diffusion(G.Grid(*shape, h=1.3), d) as op:
        assert np.array_equal(op.apply(x), port.apply(op_o, x))
        assert op.one_norm() == port.one_norm(op_o)
        u = rng.uniform(0, 1, n)
        got, info = G.step(op, u, 0.2, 9.0, 1e-9, info=True)
        want, _ = port.step(op_o, u, 0.2, 9.0, 1e-9, bnorm=info.bnorm, coln=info.coln)
        assert np.array_equal(got, want)


# ---- exponential action on the stencil ------------------------------------------------------

def test_phi1v_expmv_stencil_kats(G, kat, port):
    for i in range(int(kat["stencil.count"][0])):
        p = f"stencil.{i}"
        shape = tuple(int(v) for v in kat[p + ".shape"])
        h = float(kat[p + ".h"][0])
        x = kat[p + ".x"]
        with G.assemble_diffusion(G.Grid(*shape, h=h), kat[p + ".d"]) as op:
            got, info = G.phi1v(7.5, op, x, 1e-10, info=True)
            assert rel_l2(got, kat[p + ".phi1v"]) <= 1e-13, p
            want, log = port.phi1v(7.5, port.stencil(shape, h, kat[p + ".d"]), x, 1e-10, bnorm=info.bnorm,
                                   coln=info.coln)
            assert np.array_equal(got, want), p
            assert (info.s, info.m, info.total_terms) == (log.s, log.m, log.total_terms)
            got_e, info_e = G.expmv(7.5, op, x, 1e-10, info=True)
            # expmv has no order-dependent reduction at all: bitwise against the reference
            assert np.array_equal(got_e, kat[p + ".expmv"]), p


# ---- exponential-Euler step and run ---------------------------------------------------------

@pytest.mark.parametrize("path", ["auto", "multikernel"])
@pytest.mark.parametrize("name", RUN_NAMES)
def test_step_parity_per_step(G, port, runs_kat, name, path, monkeypatch):
    """Every step of the reference's trajectories; "auto" takes the single-cluster path on
    grids it fits, "multikernel" forces the launch sequence of the large-grid path."""
    if path == "multikernel":
        monkeypatch.setenv("GS_NO_CLUSTER", "1")
    c = case(runs_kat, name)
    grid = G.Grid(*c["shape"], h=c["h"])
    d_oracle = port.diffusion_from_labels(c["labels"])
    op_o = port.stencil(c["shape"], c["h"], d_oracle)
    with G.StencilOperator.from_labels(grid, c["labels"]) as op:
        for n in range(len(c["states"]) - 1):
            got, info = G.step(op, c["states"][n], c["rho"], c["tau"], c["tol"], info=True)
            # north_star gate: relative L2 <= 1e-10 per step vs the reference's own step
            assert rel_l2(got, c["states"][n + 1]) <= STEP_TOL, (name, n)
            # (s, m) and the terms actually used match the reference's log exactly
            assert [info.s, info.m, info.total_terms] == list(c["log"][n]), (name, n)
            # with the device's two order-dependent sums, the oracle reproduces every bit
            want, log = port.step(op_o, c["states"][n], c["rho"], c["tau"], c["tol"], bnorm=info.bnorm,
                                  coln=info.coln)
            assert np.array_equal(got, want), (name, n)
            assert info.stage_terms() == log.stage_terms()


@pytest.mark.parametrize("path", ["auto", "multikernel"])
@pytest.mark.parametrize("name", RUN_NAMES)
def test_run_parity_full(G, runs_kat, name, path, monkeypatch):
    if path == "multikernel":
        monkeypatch.setenv("GS_NO_CLUSTER", "1")
    c = case(runs_kat, name)
    steps = len(c["states"]) - 1
    grid = G.Grid(*c["shape"], h=c["h"])
    with G.StencilOperator.from_labels(grid, c["labels"]) as op:
        op.set_state(c["states"][0])
        m, infos = op.run_resident(steps, c["rho"], c["tau"], c["tol"], (0.0, 0.0, 0.0), c["center"], 0.1,
                                   metrics=True, infos=True)
        u = op.get_state()
    assert rel_l2(u, c["states"][-1]) <= RUN_TOL
    for q in range(steps):
        assert [infos[q].s, infos[q].m, infos[q].total_terms] == list(c["log"][q])
    ref_m = c["metrics"]
    for q in range(steps + 1):
        # max / min / radius are order-free reductions: exact.  The mass is a sum (tree vs serial).
        assert m[q].max_density == pytest.approx(ref_m[q, 1], rel=1e-12, abs=0)
        assert m[q].min_density == pytest.approx(ref_m[q, 2], rel=1e-12, abs=1e-300)
        assert m[q].radius == pytest.approx(ref_m[q, 3], rel=1e-12, abs=0)
        assert m[q].total_mass == pytest.approx(ref_m[q, 0], rel=1e-12)
    # node 0 sees the identical state: the order-free metrics are bitwise there
    assert m[0].max_density == ref_m[0, 1] and m[0].radius == ref_m[0, 3]


def test_seed_initial_bitwise(G, runs_kat):
    for name in RUN_NAMES:
        if name == "runmasked":
            continue
        c = case(runs_kat, name)
        cfg = G.SimConfig(seed_center=c["center"], seed_amplitude=1.0, seed_width=c["width"])
        with G.StencilOperator.from_labels(G.Grid(*c["shape"], h=c["h"]), c["labels"]) as op:
            assert np.array_equal(G.seed_initial(op, cfg, mask=True), c["states"][0]), name


def test_python_run_api_hooks(G, runs_kat):
    c = case(runs_kat, "r16")
    steps = len(c["states"]) - 1
    cfg = G.SimConfig(rho=c["rho"], exp_tol=c["tol"], nx=16, ny=16, nz=16, h=c["h"], t0=150.0,
                      t_end=150.0 + steps * c["tau"], num_steps=steps, seed_center=c["center"], snapshot_every=3)
    seen, snaps = [], []
    with G.StencilOperator.from_labels(cfg.grid(), c["labels"]) as op:
        res = G.run(cfg, op, c["states"][0], snapshot=lambda n, t, u: snaps.append((n, u)),
                    on_step=lambda m: seen.append(m.step))
    assert seen == list(range(1, steps + 1))
    assert [s[0] for s in snaps] == [0, 3, 6, 8]
    assert rel_l2(snaps[1][1], c["states"][3]) <= RUN_TOL
    assert rel_l2(res.u, c["states"][-1]) <= RUN_TOL
    assert len(res.metrics) == steps + 1


# ---- edge cases the reference tests ------------------------------------------------------------

def test_select_params_matches_reference(G, kat):
    for n, t, s, m in zip(kat["select.norm"], kat["select.tol"], kat["select.s"], kat["select.m"]):
        assert G.select_params(float(n), float(t)) == (int(s), int(m))
    with pytest.raises(ValueError):
        G.select_params(-1.0, 1e-8)
    with pytest.raises(G.NumericError):
        G.select_params(1e11, 1e-8)


def test_phi1v_edge_cases(G):
    grid = G.Grid(4, 3, 2, 1.5)
    rng = np.random.default_rng(21)
    b = rng.uniform(-1, 1, grid.num_points())
    with G.assemble_diffusion(grid, np.full(grid.num_points(), 0.1)) as op:
        assert np.array_equal(G.phi1v(0.0, op, b, 1e-10), b)                        # test_expact.cpp:212
        assert np.array_equal(G.phi1v(1.0, op, np.zeros_like(b), 1e-10), np.zeros_like(b))
        with pytest.raises(ValueError, match="vector length"):
            G.phi1v(1.0, op, np.ones(3), 1e-10)
        with pytest.raises(ValueError, match="tolerance"):
            G.phi1v(1.0, op, b, 0.0)
        assert np.array_equal(G.expmv(0.0, op, b, 1e-10), b)                        # test_expact.cpp:135
    # empty operator: phi_1(0) b = b through the small-norm branch (test_expact.cpp:218-223)
    with G.assemble_diffusion(grid, np.zeros(grid.num_points())) as zero:
        assert np.array_equal(G.phi1v(5.0, zero, b, 1e-10), b)
        assert zero.one_norm() == 0.0


def test_step_without_diffusion_is_forward_euler(G):
    """test_integrator.cpp:99-106: A = 0 -> u + tau*rho*u*(1-u) bit for bit."""
    grid = G.Grid(3, 1, 1, 1.0)
    u = np.array([0.2, 0.5, 0.9])
    rho, tau = 0.4, 0.25
    with G.assemble_diffusion(grid, np.zeros(3)) as op:
        got = G.step(op, u, rho, tau, 1e-10)
    assert np.array_equal(got, u + tau * (rho * u * (1.0 - u)))


def test_small_norm_branch(G, port):
    """|t|*||A||_1 <= 1e-8 takes b + t*A*b/2 (expact.cpp:114-122)."""
    shape = (5, 4, 3)
    d = np.full(np.prod(shape), 1e-12)
    b = np.random.default_rng(2).uniform(-1, 1, np.prod(shape))
    with G.assemble_diffusion(G.Grid(*shape, h=1.0), d) as op:
        got, info = G.phi1v(1.0, op, b, 1e-12, info=True)
        assert info.branch == 3
        want, _ = port.phi1v(1.0, port.stencil(shape, 1.0, d), b, 1e-12)
        assert np.array_equal(got, want)


def test_divergence_raises_numeric_error(G):
    """A growing operator overflows the series -> numeric_error (test_expact.cpp:140-143)."""
    shape = (4, 4, 4)
    d = np.full(64, -5.0e3)   # anti-diffusion: exponential growth
    b = np.random.default_rng(1).uniform(0, 1, 64)
    with G.assemble_diffusion(G.Grid(*shape, h=1.0), d) as op:
        with pytest.raises(G.NumericError, match="non-finite"):
            G.expmv(1e3, op, b, 1e-10)


def test_constants_preserved_by_expmv(G):
    """test_expact.cpp:108-116: rows sum to zero, so exp(tA) 1 = 1."""
    grid = G.Grid(5, 4, 3, 1.5)
    with G.assemble_diffusion(grid, np.full(grid.num_points(), 0.13)) as op:
        y = G.expmv(3.0, op, np.ones(grid.num_points()), 1e-10)
    assert np.allclose(y, 1.0, rtol=1e-12, atol=0)


@pytest.mark.parametrize("fuse", ["2", "3", "2exact", "2rerun"])
def test_mid_size_step_vs_oracle(G, port, fuse, monkeypatch):
    """64^3 phantom, several steps: bitwise against the oracle given the device sums.  The
    two-term sweeps decide on bounding maxima with an exact fallback; "2exact" runs the exact
    maxima always (GS_EXACT_MAX=1), "2rerun" takes the fallback on every sweep (=2)."""
    monkeypatch.setenv("GS_FUSE", fuse[0])
    if fuse != "2" and fuse != "3":
        monkeypatch.setenv("GS_EXACT_MAX", "1" if fuse == "2exact" else "2")
    from paper_2402_02273_b200 import phantom
    n = 64
    inten = phantom.shell_phantom(n, n, n, seed=31)
    table = np.array([port.classify(v) for v in range(256)], dtype=np.uint8)
    labels = table[inten.ravel()]
    h = 200.0 / (n - 1)
    i, j, k = phantom.pick_seed_voxel(labels, (n, n, n), 31)
    d = port.diffusion_from_labels(labels)
    u = port.seed_initial((n, n, n), h, 1.0, 1.0 / (2 * (3 * h) ** 2), (i * h, j * h, k * h), d)
    op_o = port.stencil((n, n, n), h, d)
    with G.StencilOperator.from_intensity(G.Grid(n, n, n, h), inten.ravel(), n, n, n) as op:
        assert np.array_equal(op.labels(), labels)
        for _ in range(3):
            got, info = G.step(op, u, 0.025, 33.5, 1e-8, info=True)
            want, log = port.step(op_o, u, 0.025, 33.5, 1e-8, bnorm=info.bnorm, coln=info.coln)
            assert np.array_equal(got, want)
            assert info.stage_terms() == log.stage_terms()
            ref_plain, _ = port.step(op_o, u, 0.025, 33.5, 1e-8)
            assert rel_l2(got, ref_plain) <= STEP_TOL
            u = got


@pytest.mark.parametrize("path", ["tma2", "tma2exact", "l1", "cluster"])
@pytest.mark.parametrize("tol", [0.03, 1e-3])
def test_multi_step_run_loose_tol_vs_oracle(G, port, path, tol, monkeypatch):
    """Several steps in ONE gs_run call at loose tolerances (s ~ 140, 10-16 terms per stage),
    every step bitwise against the oracle given that step's device sums.  Covers the rotating
    max slots across the steps of one launch sequence: the Taylor kernel leaves its last
    round's maxima in one slot and the update kernel zeroes all three before the next step."""
    sweep_path_env(path, monkeypatch)
    shape = (48, 32, 20) if path != "cluster" else (24, 16, 16)
    rng = np.random.default_rng(17)
    n = int(np.prod(shape))
    d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
    h = 0.25
    op_o = port.stencil(shape, h, d)
    u0 = np.zeros(n)
    u0[rng.integers(0, n, 40)] = rng.uniform(0.2, 1.0, 40)
    u0[d == 0.0] = 0.0
    k = 4
    with G.assemble_diffusion(G.Grid(*shape, h=h), d) as op:
        assert op.uses_cluster() == (path == "cluster")
        op.set_state(u0)
        _, inf = op.run_resident(k, 0.1, 33.5, tol, metrics=False, infos=True)
        got = op.get_state()
    u = u0
    for q in range(k):
        u, log = port.step(op_o, u, 0.1, 33.5, tol, bnorm=inf[q].bnorm, coln=inf[q].coln)
        assert inf[q].stage_terms() == log.stage_terms(), q
    assert np.array_equal(got, u)


# ---- both stencil sweep paths (TMA z-slab ring and the L1 fallback) on awkward shapes ------

# nx % 16 != 0 (20, 33) cannot be described by TMA: those shapes take the L1 fallback
# automatically on the "tma" parametrisations too.
TMA_SHAPES = [(48, 32, 20), (80, 40, 12), (64, 48, 1), (32, 32, 32), (16, 16, 16), (96, 17, 9), (128, 16, 3),
              (20, 12, 10), (33, 7, 5)]


SWEEP_PATHS = ["cluster", "flat2d", "tma2", "tma2exact", "tma2rerun", "tma2noxchg", "tma3", "l1"]
# 2-D shapes of the resident-tile path (gs_flat2d.cuh): ragged tiles, x extents TMA cannot
# describe, one row, one tile, C2's size
FLAT2D_SHAPES = [(64, 48, 1), (200, 190, 1), (256, 256, 1), (100, 70, 1), (33, 7, 1), (161, 1, 1), (32, 32, 1)]


def sweep_path_env(path, monkeypatch):
    """cluster: the single-cluster small-grid path; tma2: fused two-term TMA (bounding maxima,
    exact fallback); tma2exact / tma2rerun: the same with exact maxima always / the fallback
    on every sweep; tma3: fused three-term TMA; l1: the L1 single-term fallback."""
    if path != "cluster":
        monkeypatch.setenv("GS_NO_CLUSTER", "1")
    if not path.startswith("flat2d"):
        monkeypatch.setenv("GS_NO_2D", "1")
    if path == "tma2noxchg":  # atomicMax slots + grid barrier instead of the maxima exchange
        monkeypatch.setenv("GS_NO_XCHG", "1")
    if path == "l1":
        monkeypatch.setenv("GS_DISABLE_TMA", "1")
    if path == "tma3":
        monkeypatch.setenv("GS_FUSE", "3")
    if path == "tma2exact":
        monkeypatch.setenv("GS_EXACT_MAX", "1")
    if path == "tma2rerun":
        monkeypatch.setenv("GS_EXACT_MAX", "2")


# Shapes the single-cluster path takes (<= 40 K voxels, a slice of N/16 voxels at least one
# plane -- one row in 2-D): awkward x extents (not a multiple of 16), 2-D, partial planes.
CLUSTER_SHAPES = [(32, 32, 32), (16, 16, 16), (64, 48, 1), (24, 17, 16), (33, 7, 18), (20, 12, 40), (80, 16, 24),
                  (40, 30, 24), (200, 190, 1), (161, 1, 1)]
SWEEP_CASES = ([("cluster", s) for s in CLUSTER_SHAPES] + [("flat2d", s) for s in FLAT2D_SHAPES] +
               [(p, s) for p in SWEEP_PATHS if p != "cluster" and not p.startswith("flat2d") for s in TMA_SHAPES])


@pytest.mark.parametrize("path,shape", SWEEP_CASES)
def test_sweep_paths_vs_oracle(G, port, shape, path, monkeypatch):
    """Every sweep implementation (sweep_path_env) -- bitwise against the oracle."""
    sweep_path_env(path, monkeypatch)
    rng = np.random.default_rng(sum(shape))
    n = int(np.prod(shape))
    table = np.array([0.0, 0.13, 0.013, 0.05])
    d = table[rng.integers(0, 4, n)]
    h = 2.0
    op_o = port.stencil(shape, h, d)
    x = rng.uniform(-1, 1, n)
    u = rng.uniform(0, 1, n)
    with G.assemble_diffusion(G.Grid(*shape, h=h), d) as op:
        assert op.uses_cluster() == (path == "cluster"), "shape does not take the path under test"
        assert op.uses_flat2d() == path.startswith("flat2d"), "shape does not take the path under test"
        assert np.array_equal(op.apply(x), port.apply(op_o, x))
        got, info = G.step(op, u, 0.1, 33.5, 1e-9, info=True)
        want, log = port.step(op_o, u, 0.1, 33.5, 1e-9, bnorm=info.bnorm, coln=info.coln)
        assert np.array_equal(got, want)
        assert info.stage_terms() == log.stage_terms()
        got_e = G.expmv(20.0, op, x, 1e-10)
        want_e, _ = port.expmv(20.0, op_o, x, 1e-10)
        assert np.array_equal(got_e, want_e)


@pytest.mark.parametrize("path", SWEEP_PATHS)
def test_non_finite_inputs_vs_oracle(G, port, path, monkeypatch):
    """NaN and inf in the input vector on every sweep path.  The reference's norms drop NaN
    (expact.cpp:15-19), so a NaN spreads through the terms while the tests run on the rest:
    the result equals the oracle's bit for bit, NaNs in the same places.  An inf makes a
    norm infinite: numeric_error in both (expact.cpp:90-91).  On the two-term TMA path both
    cases go through the exact-maxima fallback (a non-finite key leaves the bounds open)."""
    sweep_path_env(path, monkeypatch)
    shape = (24, 16, 16) if path == "cluster" else (80, 48, 1) if path.startswith("flat2d") else (48, 32, 12)
    rng = np.random.default_rng(5)
    n = int(np.prod(shape))
    d = np.array([0.0, 0.13, 0.013, 0.05])[rng.integers(0, 4, n)]
    op_o = port.stencil(shape, 2.0, d)
    x = rng.uniform(-1, 1, n)
    x[n // 2 + 7] = np.nan
    with G.assemble_diffusion(G.Grid(*shape, h=2.0), d) as op:
        assert op.uses_cluster() == (path == "cluster")
        assert op.uses_flat2d() == path.startswith("flat2d")
        got = G.expmv(2.0, op, x, 1e-10)
        want, _ = port.expmv(2.0, op_o, x, 1e-10)
        assert np.isnan(got).any() and np.isnan(got).sum() < n
        assert np.array_equal(got, want, equal_nan=True)
        x[n // 3] = np.inf
        with pytest.raises(G.NumericError):
            G.expmv(2.0, op, x, 1e-10)
        with pytest.raises(Exception):
            port.expmv(2.0, op_o, x, 1e-10)


# ---- the C++ drop-in against the reference, called like a reference user calls it --------

@pytest.mark.parametrize("path", ["auto", "multikernel"])
def test_cpp_dropin_parity(path):
    """The C++ drop-in against the linked reference; its 24x20x16 grid takes the single-cluster
    path by default, and the multi-kernel launch sequence with GS_NO_CLUSTER=1."""
    import os
    import subprocess
    exe = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle", "_ref", "dropin_parity")
    if not os.path.exists(exe):
        pytest.skip("oracle/_ref/dropin_parity not built (needs the reference headers at build time)")
    env = dict(os.environ)
    if path == "multikernel":
        env["GS_NO_CLUSTER"] = "1"
    res = subprocess.run([exe], capture_output=True, text=True, timeout=300, env=env)
    print(res.stdout)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "all passed" in res.stdout


# ---- generic SparseOperator path: the reference's own random-operator KATs on the GPU -----

def _csr(G, kat, p):
    return G.CsrOperator(kat[p + ".offs"], kat[p + ".cols"], kat[p + ".vals"])


@pytest.mark.parametrize("tag,phi", [("expmv_rand", False), ("phi1v_rand", True), ("accept_c1", True)])
def test_csr_random_operator_kats(G, port, kat, tag, phi):
    """test_expact.cpp:79-175 / acceptance.cpp:57-86 inputs: expmv bitwise vs the reference;
    phi1v bitwise vs the oracle given the device's two sums and within 1e-12 of the reference;
    both within the reference tests' 1e-9 of the dense oracles."""
    for i in range(int(kat[tag + ".count"][0])):
        p = f"{tag}.{i}"
        t, tol, b = float(kat[p + ".t"][0]), float(kat[p + ".tol"][0]), kat[p + ".b"]
        with _csr(G, kat, p + ".A") as op:
            assert op.one_norm() == kat[p + ".A.norm1"][0], p
            if phi:
                got, info = G.phi1v(t, op, b, tol, info=True)
                want, _ = port.phi1v(t, port.csr(kat[p + ".A.offs"], kat[p + ".A.cols"], kat[p + ".A.vals"]), b, tol,
                                     bnorm=info.bnorm, coln=info.coln)
                assert np.array_equal(got, want), p
                assert rel_l2(got, kat[p + ".ref"]) <= 1e-12, p
            else:
                got = G.expmv(t, op, b, tol)
                assert np.array_equal(got, kat[p + ".ref"]), p
            dense = kat[p + ".dense"]
            assert np.max(np.abs(got - dense)) / max(np.max(np.abs(dense)), 1e-300) <= 1e-9
            if p + ".ref_exp" in kat:
                assert np.array_equal(G.expmv(t, op, b, tol), kat[p + ".ref_exp"]), p


def test_csr_apply_and_stencil_equivalence(G, kat):
    """The assembled CSR of the stencil KATs through the generic path equals the matrix-free path."""
    for i in range(int(kat["stencil.count"][0])):
        p = f"stencil.{i}"
        with _csr(G, kat, p + ".A") as op:
            assert np.array_equal(op.apply(kat[p + ".x"]), kat[p + ".Ax"]), p
            assert np.array_equal(G.expmv(7.5, op, kat[p + ".x"], 1e-10), kat[p + ".expmv"]), p


def test_csr_validation_and_errors(G):
    """SparseOperator's validation messages (sparse.cpp:14-35) and the divergence KAT
    (test_expact.cpp:140-143: a 1x1 operator 40 at t = 100 overflows)."""
    with pytest.raises(ValueError, match="not sorted unique in row 0"):
        G.CsrOperator([0, 2], [0, 0], [1.0, 2.0])
    with pytest.raises(ValueError, match="column index out of range"):
        G.CsrOperator([0, 1], [3], [1.0])
    with pytest.raises(ValueError, match="not monotone"):
        G.CsrOperator([0, 2, 1], [0, 1], [1.0, 2.0])
    with G.CsrOperator([0, 1], [0], [40.0]) as hot:
        with pytest.raises(G.NumericError, match="non-finite"):
            G.expmv(100.0, hot, np.array([1.0]), 1e-10)
    # step with an empty operator = forward Euler bit for bit (test_integrator.cpp:99-106)
    with G.CsrOperator([0, 0, 0, 0], [], []) as empty:
        u = np.array([0.2, 0.5, 0.9])
        assert np.array_equal(G.step(empty, u, 0.4, 0.25, 1e-10), u + 0.25 * (0.4 * u * (1.0 - u)))
        assert np.array_equal(G.phi1v(5.0, empty, u, 1e-10), u)


def test_csr_step_semigroup_and_linearity(G, kat):
    """expmv semigroup (test_expact.cpp:98-106) and phi1v linearity (:177-193) on the GPU."""
    p = "expmv_rand.3.A"
    with _csr(G, kat, p) as op:
        n = op.dim()
        rng = np.random.default_rng(7)
        b = rng.uniform(-1, 1, n)
        nrm = op.one_norm()
        t1, t2 = 0.8 / nrm, 1.9 / nrm
        direct = G.expmv(t1 + t2, op, b, 1e-12)
        chained = G.expmv(t2, op, G.expmv(t1, op, b, 1e-12), 1e-12)
        assert np.max(np.abs(chained - direct)) <= 1e-9 * np.max(np.abs(direct))
        b1, b2 = rng.uniform(-1, 1, n), rng.uniform(-1, 1, n)
        t = 2.0 / nrm
        lhs = G.phi1v(t, op, 0.7 * b1 - 1.3 * b2, 1e-12)
        rhs = 0.7 * G.phi1v(t, op, b1, 1e-12) - 1.3 * G.phi1v(t, op, b2, 1e-12)
        assert np.max(np.abs(lhs - rhs)) <= 1e-9 * np.max(np.abs(rhs))
