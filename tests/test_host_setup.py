"""Host logic of the product library, without a GPU (device = -1 contexts).

Integer artefacts (mesh, dof numbering, element colouring, AMG aggregates) and
the assembled mass blocks must be bit-identical to the CPU recomputation
(north star: "mesh partitioning and element colouring are bit-exact").
"""
import ctypes
import os
import re

import numpy as np
import pytest

from helpers import cube, matfree_setup, slab_reference
from oracle import pyoracle as po

import paper_1612_09447_b200 as eb

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "eqs_b200.h")).read()
    names = sorted(set(re.findall(r"^\s*(?:int|void|const char\*)\s+(eqs_\w+)\(", header, re.M)))
    assert len(names) >= 30
    lib = ctypes.CDLL(eb.eqs.LIB_PATH)
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


CASES = [cube(6), cube(10, jitter=0.1), cube(4, order=2), cube(3, jitter=0.1, order=2), matfree_setup(2, True),
         slab_reference("slab_nonlinear_rkc_spe")]


@pytest.mark.parametrize("cfg", CASES, ids=lambda c: c.get("name", "setup"))
def test_setup_artefacts_bit_exact(cfg):
    g, o = eb.FemSystem(cfg, device=-1), po.Problem(cfg)
    on, ot, orr = o.mesh()
    gn, gt, gr = g.mesh()
    assert np.array_equal(on, gn) and np.array_equal(ot, gt) and np.array_equal(orr, gr)
    oe, ofr, ofx, _ = o.dofs()
    ge, gfr, gfx = g.dofs()
    assert np.array_equal(oe, ge) and np.array_equal(ofr, gfr) and np.array_equal(ofx, gfx)
    assert np.array_equal(o.colors(), g.colors())
    for which in (0, 1):
        for a, b in zip(o.mass(which), g.mass(which)):
            assert np.array_equal(a, b)
    ol, gl = o.amg_levels(), g.amg_levels()
    assert ol == gl
    for lvl in range(len(ol) - 1):
        assert np.array_equal(o.amg_aggregates(lvl), g.amg_aggregates(lvl))


def test_config_errors_map_to_reference_classes():
    bad = cube(3)
    bad["materials"]["2"]["conductivity"]["kappa_hi"] = 1e-12  # hi < lo (materials.cpp:17-18)
    with pytest.raises(eb.ConfigError):
        eb.FemSystem(bad, device=-1)
    missing = cube(3)
    del missing["materials"]["3"]
    with pytest.raises(eb.ConfigError):
        eb.FemSystem(missing, device=-1)
    with pytest.raises(eb.ConfigError):
        eb.FemSystem("{not json", device=-1)
    unknown_set = cube(3)
    unknown_set["excitations"]["top"] = {"kind": "constant", "value": 1.0}
    with pytest.raises(eb.ConfigError):
        eb.FemSystem(unknown_set, device=-1)
    with pytest.raises(eb.ParseError):
        eb.FemSystem({**cube(3), "mesh": {"file": "/nonexistent.msh"}}, device=-1)
    trunc = cube(3)
    for bad_t in (1.5, [0.1, 1.5], "x"):  # additive key: per-level thresholds in [0, 1), or 0
        trunc["solver"]["amg_vcycle_truncate"] = bad_t
        with pytest.raises(eb.ConfigError):
            eb.FemSystem(trunc, device=-1)


def test_vcycle_truncation_keeps_the_reference_hierarchy():
    """solver.amg_vcycle_truncate changes only the V-cycle's
    copy of P_1 and the coarser Galerkin operators: the hierarchy a context
    reports stays the reference algorithm's, bit for bit."""
    cfg = cube(10, jitter=0.1)
    off = dict(cfg, solver=dict(cfg["solver"], amg_vcycle_truncate=0.0))
    g_on, g_off = eb.FemSystem(cfg, device=-1), eb.FemSystem(off, device=-1)
    assert g_on.amg_levels() == g_off.amg_levels()
    for lvl in range(len(g_on.amg_levels())):
        for which in (0, 1, 2):
            if lvl + 1 == len(g_on.amg_levels()) and which > 0:
                continue
            a, b = g_on.amg_level_csr(lvl, which), g_off.amg_level_csr(lvl, which)
            assert all(np.array_equal(x, y) for x, y in zip(a, b))
    with pytest.raises(eb.InvalidArgument):
        c = cube(3)
        c["mesh"]["box"]["z_planes"] = [1.5, 2.0]
        eb.FemSystem(c, device=-1)


def test_host_only_context_refuses_compute():
    g = eb.FemSystem(cube(3), device=-1)
    with pytest.raises(eb.CudaError):
        g.eval_rhs(0.0, np.zeros(g.n_free))


def test_lift_full_matches_oracle():
    cfg = slab_reference("slab_nonlinear_rkc_spe")
    g, o = eb.FemSystem(cfg, device=-1), po.Problem(cfg)
    x = po.random_vec(g.n_free, 4)
    for t in (0.0, 3.7e-3):
        assert np.array_equal(g.lift_full(t, x), o.lift_full(t, x))


def test_msh_roundtrip_loads_same_mesh(tmp_path):
    """load_msh (msh_io.cpp:63-175): a box written as MSH 2.2 loads to the same arrays."""
    cfg = cube(3, jitter=0.1)
    o = po.Problem(cfg)
    nodes, tets, region = o.mesh()
    _, _, fx, fs = o.dofs()
    path = tmp_path / "box.msh"
    with open(path, "w") as f:
        f.write("$MeshFormat\n2.2 0 8\n$EndMeshFormat\n")
        f.write('$PhysicalNames\n2\n2 1 "ground"\n2 2 "hv"\n$EndPhysicalNames\n')
        f.write(f"$Nodes\n{len(nodes)}\n")
        for i, p in enumerate(nodes):
            f.write(f"{i + 1} {float(p[0])!r} {float(p[1])!r} {float(p[2])!r}\n")
        f.write("$EndNodes\n")
        z = nodes[:, 2]
        tris = []
        for tag, zz in ((1, 0.0), (2, 1.0)):
            for t in tets:
                on = [v for v in t if abs(z[v] - zz) < 1e-12]
                if len(on) == 3:
                    tris.append((tag, on))
        f.write(f"$Elements\n{len(tris) + len(tets)}\n")
        eid = 0
        for tag, on in tris:
            eid += 1
            f.write(f"{eid} 2 2 {tag} {tag} {on[0] + 1} {on[1] + 1} {on[2] + 1}\n")
        for t, r in zip(tets, region):
            eid += 1
            f.write(f"{eid} 4 2 {r} {r} {t[0] + 1} {t[1] + 1} {t[2] + 1} {t[3] + 1}\n")
        f.write("$EndElements\n")
    file_cfg = dict(cfg)
    file_cfg["mesh"] = {"file": str(path)}
    g, o2 = eb.FemSystem(file_cfg, device=-1), po.Problem(file_cfg)
    gn, gt, gr = g.mesh()
    assert np.array_equal(gn, nodes) and np.array_equal(gt, tets) and np.array_equal(gr, region)
    assert np.array_equal(g.colors(), o2.colors())
    for a, b in zip(o2.mass(0), g.mass(0)):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("cfg", [cube(10, jitter=0.1), cube(3, jitter=0.1, order=2),
                                 slab_reference("slab_nonlinear_rkc_spe")], ids=lambda c: c.get("name", "setup"))
def test_amg_hierarchy_values_bit_exact(cfg):
    """Galerkin hierarchy A_l, P_l, R_l (amg.cpp:90-143) of the host setup
    (row-parallel SpGEMM) == the oracle's, bit for bit."""
    g, o = eb.FemSystem(cfg, device=-1), po.Problem(cfg)
    n_levels = len(o.amg_levels())
    for lvl in range(n_levels):
        for which in ((0, 1, 2) if lvl + 1 < n_levels else (0,)):
            a, b = po.amg_level_csr(o, lvl, which), g.amg_level_csr(lvl, which)
            assert a[:2] == b[:2]
            for x, y in zip(a[2:], b[2:]):
                assert np.array_equal(x, y), (lvl, which)


@pytest.mark.skipif(not os.path.isdir("/root/reference/proj/include"), reason="reference headers absent")
def test_cpp_shim_compiles_against_reference_headers():
    """integration/eqs_gpu_shim.hpp (the INTEGRATION.md shim) compiles against
    the unmodified reference headers and include/eqs_b200.h."""
    import subprocess
    import sysconfig
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    site = sysconfig.get_paths()["purelib"]
    src = '#include "eqs_gpu_shim.hpp"\nint main() { return 0; }\n'
    cmd = ["g++", "-std=c++20", "-fsyntax-only", "-Wall", "-Wextra", "-Werror", "-x", "c++", "-",
           "-I" + os.path.join(root, "integration"), "-I" + os.path.join(root, "oracle", "ref_shim"),
           "-I/root/reference/proj/include", "-I" + os.path.join(root, "include"),
           "-I" + os.path.join(site, "include", "cudnn_frontend", "thirdparty")]
    r = subprocess.run(cmd, input=src, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
