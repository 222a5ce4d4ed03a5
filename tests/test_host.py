"""CPU-side checks: the C-ABI library loads and exports every declared symbol, the
host-side API logic, and the phantom generator.  No compute calls need a GPU here."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "gliosim_b200.h")).read()
    return sorted(set(re.findall(r"^\S.*?\b(gs_[a-z0-9_]+)\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def lib_path():
    from paper_2402_02273_b200 import build
    return build.build()


def test_library_exports_every_declared_symbol(lib_path):
    out = subprocess.run(["nm", "-D", "--defined-only", lib_path], capture_output=True, text=True, check=True).stdout
    exported = set(re.findall(r"\bT (gs_[a-z0-9_]+)$", out, flags=re.M))
    decl = declared_symbols()
    assert len(decl) >= 20
    missing = [s for s in decl if s not in exported]
    assert not missing, missing


def test_library_loads_and_binds(lib_path):
    from paper_2402_02273_b200 import _native
    lib = _native.load()
    for name in declared_symbols():
        assert hasattr(lib, name)
    assert set(_native.EXPORTS) == set(declared_symbols())


def test_library_targets_sm100a(lib_path):
    out = subprocess.run(["cuobjdump", "--list-elf", lib_path], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_gpu_fails_loudly(lib_path):
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2402_02273_b200 import gliosim as G
    with pytest.raises(G.CudaError):
        G.StencilOperator(G.Grid(4, 4, 4, 1.0))


def test_select_params_host_side_matches_reference(lib_path, kat):
    from paper_2402_02273_b200 import gliosim as G
    for n, t, s, m in zip(kat["select.norm"], kat["select.tol"], kat["select.s"], kat["select.m"]):
        assert G.select_params(float(n), float(t)) == (int(s), int(m))


def test_grid_and_config_validation():
    from paper_2402_02273_b200 import gliosim as G
    with pytest.raises(ValueError, match="point counts"):
        G.Grid(0, 1, 1, 1.0)
    with pytest.raises(ValueError, match="spacing"):
        G.Grid(1, 1, 1, 0.0)
    cfg = G.SimConfig()
    cfg.validate()
    assert cfg.tau() == 33.5
    cfg.rho = -1
    with pytest.raises(G.DataError, match="'rho'"):
        cfg.validate()
    cfg = G.SimConfig(num_steps=100)
    assert G.time_at(cfg, 100) == 3500.0 and G.time_at(cfg, 0) == 150.0


def test_phantom_is_deterministic_and_banded(port):
    from paper_2402_02273_b200 import phantom
    a = phantom.shell_phantom(32, 28, 24, seed=9)
    b = phantom.shell_phantom(32, 28, 24, seed=9)
    assert np.array_equal(a, b)
    assert not np.array_equal(a, phantom.shell_phantom(32, 28, 24, seed=10))
    table = np.array([port.classify(v) for v in range(256)], dtype=np.uint8)
    labels = table[a.ravel()]
    counts = np.bincount(labels, minlength=4)
    assert all(counts > 0)  # air, white, gray, skull all present
    # air carries no noise
    assert set(np.unique(a[a < 2])) <= {0}
    i, j, k = phantom.pick_seed_voxel(labels, (32, 28, 24), 9)
    assert labels[i + 32 * (j + 28 * k)] == 1


def test_workloads_describe_baseline_configs():
    from paper_2402_02273_b200 import workloads as W
    names = [w.name for w in W.CONFIGS]
    assert names == ["C1", "C2", "C3", "C4", "C5"]
    c4 = W.get("C4")
    assert (c4.nx, c4.ny, c4.nz, c4.steps) == (256, 256, 256, 100)
    assert c4.tau == 33.5


def test_cpp_header_compiles_standalone(tmp_path):
    """include/gliosim_b200.hpp needs nothing but the C-ABI header (no reference headers)."""
    src = tmp_path / "t.cpp"
    src.write_text('#include "gliosim_b200.hpp"\n'
                   'struct G { int nx = 4, ny = 4, nz = 4; double h = 1.0; };\n'
                   'struct D { G grid; std::vector<double> d = std::vector<double>(64, 0.1); };\n'
                   'int main() { D d; (void)&gliosim_b200::assemble_diffusion<D>; return 0; }\n')
    subprocess.run(["g++", "-std=c++17", "-fsyntax-only", "-I", os.path.join(ROOT, "include"), str(src)], check=True)
