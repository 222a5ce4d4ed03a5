"""File formats against the reference, byte for byte.

* Golden files written by the unmodified reference (tests/golden/make_io_golden.py) pin
  write_vtk / write_metrics_csv / write_label_volume output.
* Where oracle/_ref is built (this container), every reader and writer is also compared
  with the reference live: identical bytes, identical values, identical error messages on
  fuzzed inputs (truncations and byte mutations of valid files).
* The cases of the reference's own suites (test_io.cpp, test_imaging.cpp) are restated.
No GPU needed: these are host functions of the native library.
"""
import os

import numpy as np
import pytest

from paper_2402_02273_b200 import gliosim as G

IO = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "io")


def slurp(p):
    with open(p, "rb") as f:
        return f.read()


def spit(p, data):
    with open(p, "wb") as f:
        f.write(data if isinstance(data, bytes) else data.encode())


def outcome_ours(fn):
    try:
        return ("ok", fn())
    except G.DataError as e:
        return ("data_error", str(e))
    except ValueError as e:
        return ("invalid_argument", str(e))


def outcome_ref(fn):
    from oracle import OracleError
    try:
        return ("ok", fn())
    except OracleError as e:
        kind = {1: "invalid_argument", 3: "data_error"}.get(e.code, f"code{e.code}")
        return (kind, str(e).split(": ", 1)[1])


# ---- write_vtk ---------------------------------------------------------------------------

def test_snapshot_layout_is_exactly_the_documented_one(tmp_path):
    """test_io.cpp:51-69."""
    p = tmp_path / "layout.vtk"
    G.write_vtk(G.ScalarField(G.Grid(2, 2, 1, 1.5), np.array([0.0, 0.5, 0.25, 1.0])), p)
    want = ("# vtk DataFile Version 3.0\ntumor density snapshot\nASCII\nDATASET STRUCTURED_POINTS\n"
            "DIMENSIONS 2 2 1\nSPACING 1.5 1.5 1.5\nORIGIN 0 0 0\nPOINT_DATA 4\n"
            "SCALARS tumor_density float 1\nLOOKUP_TABLE default\n0\n0.5\n0.25\n1\n")
    assert slurp(p).decode() == want
    assert slurp(p) == slurp(os.path.join(IO, "layout.vtk"))


def test_snapshot_bytes_match_reference_golden_with_labels(tmp_path):
    vals = np.load(os.path.join(IO, "mixed_values.npy"))
    labels = np.load(os.path.join(IO, "mixed_labels.npy"))
    p = tmp_path / "mixed.vtk"
    G.write_vtk(G.ScalarField(G.Grid(3, 4, 2, 200.0 / 49.0, (1.0, -2.0, 0.125)), vals), p, labels)
    assert slurp(p) == slurp(os.path.join(IO, "mixed.vtk"))


def test_snapshot_round_trips_doubles_bit_for_bit(tmp_path):
    """test_io.cpp:71-91."""
    g = G.Grid(3, 4, 2, 200.0 / 49.0, (1.0, -2.0, 0.125))
    rng = np.random.default_rng(17)
    u = rng.uniform(-1, 1, g.num_points())
    u[:3] = [1.0 / 3.0, 1e-17, 0.1]
    p = tmp_path / "rt.vtk"
    G.write_vtk(G.ScalarField(g, u), p)
    back = G.read_vtk(p)
    assert (back.grid.nx, back.grid.ny, back.grid.nz) == (3, 4, 2)
    assert back.grid.h == g.h and back.grid.origin == g.origin
    assert np.array_equal(back.values.view(np.uint64), u.view(np.uint64))


def test_same_field_twice_gives_identical_files(tmp_path):
    """test_io.cpp:93-105."""
    u = G.ScalarField(G.Grid(4, 3, 2, 0.7), np.random.default_rng(29).uniform(0, 1, 24))
    G.write_vtk(u, tmp_path / "a.vtk")
    G.write_vtk(u, tmp_path / "b.vtk")
    assert slurp(tmp_path / "a.vtk") == slurp(tmp_path / "b.vtk")


def test_material_labels_ride_along_and_readers_skip_them(tmp_path):
    """test_io.cpp:107-122."""
    p = tmp_path / "m.vtk"
    u = G.ScalarField(G.Grid(2, 2, 1, 1.0), np.array([0.1, 0.2, 0.3, 0.4]))
    G.write_vtk(u, p, G.MaterialVolume(u.grid, np.array([0, 1, 2, 3], dtype=np.uint8)))
    text = slurp(p).decode()
    assert "SCALARS material int 1\n" in text and "0\n1\n2\n3\n" in text
    assert np.array_equal(G.read_vtk(p).values, u.values)


def test_writer_argument_errors(tmp_path):
    with pytest.raises(ValueError, match="field length does not match its grid"):
        G.write_vtk(G.ScalarField(G.Grid(2, 2, 1, 1.0), np.zeros(3)), tmp_path / "x.vtk")
    with pytest.raises(ValueError, match="material volume does not match the field grid"):
        G.write_vtk(G.ScalarField(G.Grid(2, 2, 1, 1.0), np.zeros(4)), tmp_path / "x.vtk", np.zeros(3, np.uint8))
    with pytest.raises(G.DataError, match="cannot open .* for writing"):
        G.write_vtk(G.ScalarField(G.Grid(2, 2, 1, 1.0), np.zeros(4)), tmp_path / "no" / "x.vtk")


def _stress_values(n, seed):
    rng = np.random.default_rng(seed)
    parts = [
        rng.uniform(0, 1, n // 4),                                    # densities
        rng.uniform(0, 1, n // 8) * 10.0 ** rng.integers(-320, -4, n // 8),  # far-field tails
        rng.standard_normal(n // 8) * 10.0 ** rng.integers(-30, 30, n // 8),
        rng.integers(-(10 ** 6), 10 ** 6, n // 8).astype(np.float64),  # integers
        np.frombuffer(rng.bytes(8 * (n // 4)), dtype=np.float64),   # arbitrary bit patterns
    ]
    v = np.concatenate(parts)
    v = v[np.isfinite(v)]
    return np.resize(v, n)


def test_parallel_formatter_matches_printf_exactly(tmp_path):
    """The multi-threaded exact %.17g path (several 32K-value blocks) against Python's
    correctly rounded '%.17g' (the same digits glibc prints for every finite double)."""
    n = 40 * 40 * 60
    v = _stress_values(n, 3)
    p = tmp_path / "big.vtk"
    G.write_vtk(G.ScalarField(G.Grid(40, 40, 60, 0.25), v), p, threads=8)
    lines = slurp(p).decode().split("\n")
    body = lines[10:10 + n]

    def c17(x):
        s = "%.17g" % x
        return s

    want = [c17(x) for x in v]
    bad = [(i, a, b) for i, (a, b) in enumerate(zip(body, want)) if a != b]
    assert not bad, bad[:5]
    # thread count never changes the bytes
    p1 = tmp_path / "one.vtk"
    G.write_vtk(G.ScalarField(G.Grid(40, 40, 60, 0.25), v), p1, threads=1)
    assert slurp(p1) == slurp(p)


def test_writer_matches_reference_live(ref, tmp_path):
    for seed, shape in [(1, (5, 7, 3)), (2, (64, 32, 20)), (3, (1, 1, 1))]:
        n = shape[0] * shape[1] * shape[2]
        v = _stress_values(n, seed)
        lab = np.random.default_rng(seed).integers(0, 4, n).astype(np.uint8)
        origin = (-3.5, 0.1, 1e-3 * seed)
        h = 200.0 / (shape[0] + 6)
        for labels in (None, lab):
            a, b = tmp_path / "ours.vtk", tmp_path / "ref.vtk"
            G.write_vtk(G.ScalarField(G.Grid(*shape, h, origin), v), a, labels)
            ref.write_vtk(b, v, shape, h, origin, labels)
            assert slurp(a) == slurp(b), (seed, shape, labels is None)


# ---- read_vtk ----------------------------------------------------------------------------

@pytest.mark.parametrize("mutate,needle", [
    (lambda t: "bogus\n" + t, "missing '# vtk DataFile'"),
    (lambda t: t.replace("ASCII", "BINARY", 1), "expected 'ASCII', found 'BINARY'"),
    (lambda t: t.replace("DIMENSIONS 2 2 1", "DIMENSIONS 0 2 1", 1), "positive integer"),
    (lambda t: t.replace("SPACING 1 1 1", "SPACING 1 2 1", 1), "isotropic"),
    (lambda t: t.replace("POINT_DATA 4", "POINT_DATA 5", 1), "disagrees with DIMENSIONS"),
    (lambda t: t.replace("0.375", "oops", 1), "expected a number"),
    (lambda t: t[:-5], "unexpected end of file"),
])
def test_reader_rejects_malformed_snapshots(tmp_path, mutate, needle):
    """test_io.cpp:124-175."""
    p = tmp_path / "broken.vtk"
    G.write_vtk(G.ScalarField(G.Grid(2, 2, 1, 1.0), np.array([0.125, 0.25, 0.375, 0.5])), p)
    spit(p, mutate(slurp(p).decode()))
    with pytest.raises(G.DataError, match=None) as ei:
        G.read_vtk(p)
    assert needle in str(ei.value)


def test_reader_missing_file(tmp_path):
    with pytest.raises(G.DataError, match="cannot open"):
        G.read_vtk(tmp_path / "nothere.vtk")


def test_reader_matches_reference_on_fuzzed_files(ref, tmp_path):
    """Truncations at every byte and random single-byte mutations of valid snapshots:
    same values or the same error message as the reference's read_vtk."""
    rng = np.random.default_rng(11)
    base = tmp_path / "base.vtk"
    G.write_vtk(G.ScalarField(G.Grid(2, 3, 2, 0.5, (1.0, 2.0, -3.0)), rng.uniform(-1, 1, 12)), base,
                np.arange(12, dtype=np.uint8) % 4)
    good = slurp(base)
    variants = [good[:k] for k in range(len(good) + 1)]
    alphabet = b"0123456789.-+eE \n\tx#"
    for _ in range(600):
        b = bytearray(good)
        for _ in range(int(rng.integers(1, 3))):
            b[int(rng.integers(0, len(b)))] = alphabet[int(rng.integers(0, len(alphabet)))]
        variants.append(bytes(b))
    variants += [good.replace(b"0.5 0.5 0.5", b"inf inf inf"), good.replace(b"POINT_DATA 12", b"POINT_DATA +12"),
                 good.replace(b"DIMENSIONS 2", b"DIMENSIONS 99999999999"), good.replace(b"ASCII", b"ASCII\n\n\n"),
                 good.replace(b"ORIGIN 1", b"ORIGIN 0x1p3"), good.replace(b"ORIGIN 1", b"ORIGIN 1e-400")]
    p = tmp_path / "f.vtk"
    mism = []
    for v in variants:
        spit(p, v)
        o = outcome_ours(lambda: G.read_vtk(p))
        r = outcome_ref(lambda: ref.read_vtk(p))
        if o[0] == "ok" and r[0] == "ok":
            f = o[1]
            dims, h, origin, vals = r[1]
            same = ((f.grid.nx, f.grid.ny, f.grid.nz) == dims and f.grid.h == h and tuple(f.grid.origin) == origin
                    and np.array_equal(f.values.view(np.uint64), vals.view(np.uint64)))
            if not same:
                mism.append((v, "values"))
        elif o != r:
            mism.append((v, o, r))
    assert not mism, mism[:3]


def test_subnormal_values_follow_the_reference_reader(ref):
    """The reference's stod rejects underflowing tokens (ERANGE); so must we."""
    p = os.path.join(IO, "mixed.vtk")
    assert outcome_ours(lambda: G.read_vtk(p))[0] == outcome_ref(lambda: ref.read_vtk(p))[0]
    o, r = outcome_ours(lambda: G.read_vtk(p)), outcome_ref(lambda: ref.read_vtk(p))
    if o[0] != "ok":
        assert o == r


# ---- metrics csv -------------------------------------------------------------------------

def test_metrics_csv_flat_layout(tmp_path):
    """test_io.cpp:177-206."""
    p = tmp_path / "m.csv"
    G.write_metrics_csv([], p)
    assert slurp(p) == b"step,time_days,total_mass,max_density,radius_mm\n"
    a = G.StepMetrics(0, 150.0, 2.5, 0.0625, -0.5, 0.0)
    b = G.StepMetrics(1, 183.5, 3.0625, 0.125, 0.0, 12.5)
    G.write_metrics_csv([a, b], p)
    assert slurp(p) == (b"step,time_days,total_mass,max_density,radius_mm\n"
                        b"0,150,2.5,0.0625,0\n1,183.5,3.0625,0.125,12.5\n")


def test_metrics_csv_matches_reference_golden(tmp_path):
    z = np.load(os.path.join(IO, "metrics_series.npz"))
    series = [G.StepMetrics(int(s), float(t), *map(float, m)) for s, t, m in zip(z["steps"], z["times"], z["m4"])]
    p = tmp_path / "m.csv"
    G.write_metrics_csv(series, p)
    assert slurp(p) == slurp(os.path.join(IO, "metrics.csv"))


# ---- PGM stacks, raw and label volumes ---------------------------------------------------

def pgm(w, h, pix, header=None):
    head = header if header is not None else f"P5\n# a comment\n{w} {h}\n255\n"
    return head.encode() + bytes(pix)


def test_load_stack_reads_pgm_slices_bottom_first(tmp_path):
    """test_imaging.cpp: P5 slices with comments; intensity (x,y,z) at x + y*w + z*w*h."""
    rng = np.random.default_rng(4)
    sl = [rng.integers(0, 256, 6 * 5).astype(np.uint8) for _ in range(3)]
    paths = []
    for i, s in enumerate(sl):
        p = tmp_path / f"s{i}.pgm"
        spit(p, pgm(6, 5, s, "P5 #c\n6 #w\n5\n#x\n255 " if i == 1 else None))
        paths.append(p)
    st = G.load_stack(paths)
    assert (st.width, st.height, st.num_slices) == (6, 5, 3)
    assert np.array_equal(st.intensities, np.concatenate(sl))
    assert st.at(2, 3, 1) == sl[1][2 + 3 * 6]


def test_loader_errors(tmp_path):
    p = tmp_path / "a.pgm"
    cases = [
        (b"P2\n2 2\n255\n" + bytes(4), "magic is 'P2', expected P5"),
        (b"P5\n2 2\n65535\n" + bytes(8), "maxval 65535, expected 255"),
        (b"P5\n2 x\n255\n", "bad height 'x'"),
        (b"P5\n2 2\n255\n" + bytes(3), "truncated pixel data"),
        (b"P5\n2 2", "truncated header"),
    ]
    for data, needle in cases:
        spit(p, data)
        with pytest.raises(G.DataError) as ei:
            G.load_stack([p])
        assert needle in str(ei.value), (data, str(ei.value))
    with pytest.raises(G.DataError, match="no slice files given"):
        G.load_stack([])
    with pytest.raises(G.DataError, match="cannot open"):
        G.load_stack([tmp_path / "missing.pgm"])
    spit(tmp_path / "b.pgm", pgm(3, 2, bytes(6)))
    spit(p, pgm(2, 2, bytes(4)))
    with pytest.raises(G.DataError, match="is 3x2, previous slices are 2x2"):
        G.load_stack([p, tmp_path / "b.pgm"])


def test_loaders_match_reference_on_fuzzed_files(ref, tmp_path):
    rng = np.random.default_rng(21)
    good_pgm = pgm(4, 3, rng.integers(0, 256, 12).astype(np.uint8), "P5\n#c\n4 3\n255\n")
    good_raw = b"4 3 2\n" + bytes(rng.integers(0, 256, 24).astype(np.uint8))
    alphabet = b"0123456789 \n\t#P5x-+"
    mism = []
    for good, kind in ((good_pgm, "pgm"), (good_raw, "raw")):
        variants = [good[:k] for k in range(len(good) + 1)]
        for _ in range(300):
            b = bytearray(good)
            pos = int(rng.integers(0, min(len(b), 16)))
            b[pos] = alphabet[int(rng.integers(0, len(alphabet)))]
            variants.append(bytes(b))
        variants += [good + b"extra"]
        p = tmp_path / f"f.{kind}"
        for v in variants:
            spit(p, v)
            if kind == "pgm":
                o = outcome_ours(lambda: G.load_stack([p]))
                r = outcome_ref(lambda: ref.load_stack([p]))
                if o[0] == "ok" and r[0] == "ok":
                    st = o[1]
                    if (st.width, st.height, st.num_slices) != r[1][0] or not np.array_equal(st.intensities, r[1][1]):
                        mism.append((v, "values"))
                    continue
            else:
                o = outcome_ours(lambda: G.load_raw_volume(p))
                r = outcome_ref(lambda: ref.load_raw_volume(p))
                if o[0] == "ok" and r[0] == "ok":
                    st = o[1]
                    if (st.width, st.height, st.num_slices) != r[1][0] or not np.array_equal(st.intensities, r[1][1]):
                        mism.append((v, "values"))
                    continue
            if o != r:
                mism.append((v, o, r))
    assert not mism, mism[:3]


def test_raw_volume_header_errors(tmp_path):
    p = tmp_path / "v.raw"
    for data, needle in [(b"", "missing header"), (b"2 2\n" + bytes(4), "bad header '2 2'"),
                         (b"2 2 1 7\n" + bytes(4), "trailing header token '7'"),
                         (b"2 2 1\n" + bytes(3), "truncated voxel data"), (b"0 2 1\n", "bad header")]:
        spit(p, data)
        with pytest.raises(G.DataError) as ei:
            G.load_raw_volume(p)
        assert needle in str(ei.value)


def test_label_volume_round_trip_and_golden(tmp_path):
    lab = np.load(os.path.join(IO, "labels.npy"))
    g = G.Grid(5, 4, 3, 1.0)
    p = tmp_path / "l.raw"
    G.write_label_volume(G.MaterialVolume(g, lab), p)
    assert slurp(p) == slurp(os.path.join(IO, "labels.raw"))
    assert np.array_equal(G.read_label_volume(p, g).labels, lab)
    with pytest.raises(G.DataError, match=r"is 5x4x3, grid wants 5x4x4"):
        G.read_label_volume(p, G.Grid(5, 4, 4, 1.0))
    bad = bytearray(slurp(p))
    bad[-1] = 7
    spit(p, bytes(bad))
    with pytest.raises(G.DataError, match="byte 7 is not a material label"):
        G.read_label_volume(p, g)


def test_label_volume_matches_reference(ref, tmp_path):
    lab = np.random.default_rng(2).integers(0, 4, 7 * 6 * 5).astype(np.uint8)
    a, b = tmp_path / "a.raw", tmp_path / "b.raw"
    G.write_label_volume(G.MaterialVolume(G.Grid(7, 6, 5, 1.0), lab), a)
    ref.write_label_volume(b, lab, (7, 6, 5))
    assert slurp(a) == slurp(b)
    assert np.array_equal(ref.read_label_volume(a, (7, 6, 5)), G.read_label_volume(b, G.Grid(7, 6, 5, 1.0)).labels)
    bad = bytearray(slurp(a))
    bad[20] = 200
    spit(a, bytes(bad))
    o = outcome_ours(lambda: G.read_label_volume(a, G.Grid(7, 6, 5, 1.0)))
    r = outcome_ref(lambda: ref.read_label_volume(a, (7, 6, 5)))
    assert o == r and o[0] == "data_error"
