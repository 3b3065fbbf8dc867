"""CPU checks of the drop-in boundary: the C-ABI library loads, exports every
entry point include/b200hydro.h declares, and the host-side setup (basis tables,
cartesian restriction indices, box mask) is bit-identical to the reference."""

import ctypes
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden

HEADER = os.path.join(ROOT, "include", "b200hydro.h")


def header_functions():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(hx_\w+)\s*\(", text, re.M)))


def test_library_built_and_exports_header_symbols():
    from paper_2112_07075_b200 import _lib

    assert os.path.exists(_lib.LIB_PATH), "run `python -m paper_2112_07075_b200.build`"
    lib = ctypes.CDLL(_lib.LIB_PATH)
    declared = header_functions()
    assert len(declared) >= 20
    for name in declared:
        assert hasattr(lib, name), f"{name} declared in b200hydro.h but not exported"
    # the ctypes binding covers exactly the header
    assert set(_lib.exported_symbols()) == set(declared)


def test_library_is_sm100a():
    from paper_2112_07075_b200 import _lib

    import subprocess

    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", _lib.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_product_fails_loudly_without_cuda():
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    from paper_2112_07075_b200 import _lib
    from paper_2112_07075_b200.fespace import cartesian_mesh, compute_geometric_factors
    from paper_2112_07075_b200.tensor_basis import gauss_legendre

    mesh = cartesian_mesh(2, (1.0, 1.0), (2, 2), 2)
    with pytest.raises(_lib.BackendUnavailable):
        compute_geometric_factors(mesh, gauss_legendre(4))


def test_host_basis_tables_bitwise():
    from paper_2112_07075_b200.tensor_basis import eval_basis, gauss_legendre, gauss_lobatto_nodes

    g = golden("basis")
    for p in range(1, 5):
        q = gauss_legendre(p + 2)
        assert np.array_equal(q.points, g[f"qpts_{p}"]) and np.array_equal(q.weights, g[f"qw_{p}"])
        b = eval_basis(gauss_lobatto_nodes(p), q)
        assert np.array_equal(b.B, g[f"B_{p}"]) and np.array_equal(b.G, g[f"G_{p}"])
        tn = np.zeros(1) if p == 1 else gauss_lobatto_nodes(p - 1)
        bt = eval_basis(tn, q)
        assert np.array_equal(bt.B, g[f"Bt_{p}"])


def test_cartesian_restriction_indices_bitwise():
    from paper_2112_07075_b200.fespace import cartesian_mesh

    g = golden("mesh")
    i = 0
    while f"dofmap_{i}" in g:
        case = g[f"case_{i}"]
        d, p = int(case[0]), int(case[1])
        counts = tuple(int(c) for c in case[2 : 2 + d])
        m = cartesian_mesh(d, (1.0,) * d, counts, p)
        assert np.array_equal(m.node_dofmap, g[f"dofmap_{i}"])
        assert np.array_equal(m.coords, g[f"coords_{i}"])
        i += 1


@pytest.mark.parametrize("d,p", [(2, 2), (3, 1), (3, 3)])
def test_boundary_nodes_and_mask(d, p):
    from oracle import pa_oracle as O
    from paper_2112_07075_b200.fespace import cartesian_mesh
    from paper_2112_07075_b200.hydro import box_velocity_bc

    m = cartesian_mesh(d, (1.0,) * d, (3,) * d, p)
    on_edge = np.any((m.coords < 1e-12) | (m.coords > 1 - 1e-12), axis=1)
    assert np.array_equal(np.sort(m.boundary_nodes()), np.flatnonzero(on_edge))
    assert np.array_equal(box_velocity_bc(m), O.box_mask(m.coords))
