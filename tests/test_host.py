"""CPU-side checks of the product's host code: mesh / basis setup is
bit-identical to the reference's (golden), the L->E transpose map gives the
np.add.at order, and the C-ABI library exports every declared symbol."""

import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden_names, load_golden

import paper_2205_12721_b200 as P
from paper_2205_12721_b200 import _lib


@pytest.mark.parametrize("name", golden_names("op"))
def test_host_setup_is_bitwise_reference(name):
    g = load_golden(name)
    dim, order, nq = int(g["dim"]), int(g["order"]), int(g["n_quad"])
    mesh = P.build_box(dim, tuple(int(c) for c in g["counts"]), order)
    assert np.array_equal(mesh.restriction, g["restriction"])
    assert mesh.restriction.dtype == np.int32
    assert np.array_equal(mesh.fixed_mask, g["fixed"])
    assert np.array_equal(mesh.coords, g["coords"])
    em = P.build_eval_matrices(P.Basis1D.gauss_lobatto(order), P.gauss_legendre_1d(nq))
    assert np.array_equal(em.b, g["B"])
    assert np.array_equal(em.g, g["G"])
    assert np.array_equal(P.tensor_weights(P.gauss_legendre_1d(nq), dim), g["wq"])


def test_kershaw_bitwise_reference():
    g = load_golden("kershaw_6x2x2_p2")
    mesh = P.apply_kershaw(P.build_cartesian(P.MeshSpec(3, 6, 2, 2, order=2)), 0.3, 0.3)
    assert np.array_equal(mesh.coords, g["coords"])


def test_mesh_spec_validation():
    with pytest.raises(P.MeshConfigError):
        P.MeshSpec(3, 5, 2, 2).validate()
    with pytest.raises(P.MeshConfigError):
        P.build_box(3, (2, 2), 1)
    with pytest.raises(ValueError):
        P.gauss_legendre_1d(0)


def test_l2e_map_reproduces_add_at_order():
    from paper_2205_12721_b200.operator import DeviceMesh
    rng = np.random.default_rng(0)
    mesh = P.build_box(3, (3, 2, 2), 2)
    dm = DeviceMesh(mesh, "cpu")
    off = dm.l2e_offsets.numpy()
    idx = dm.l2e_index.numpy().view(np.uint32)
    np_ = mesh.restriction.shape[1]
    E = rng.standard_normal(mesh.restriction.shape)
    want = np.zeros(mesh.n_nodes)
    np.add.at(want, mesh.restriction.ravel(), E.ravel())
    got = np.zeros(mesh.n_nodes)
    for node in range(mesh.n_nodes):
        acc = 0.0
        ents = idx[off[node]:off[node + 1]]
        assert np.all(np.diff(ents // np_) > 0)        # ascending element order
        for u in ents:
            acc += E[u // np_, u % np_]
        got[node] = acc
    assert np.array_equal(got, want)                   # same order => bitwise equal
    flags = dm.fixed.numpy()
    assert flags.size % 4 == 0 and not flags[mesh.n_nodes:].any()   # padded to whole 32-bit words
    flags = flags[:mesh.n_nodes]
    for a in range(3):
        assert np.array_equal(((flags >> a) & 1).astype(bool), mesh.fixed_mask[a])


def test_library_exports_every_declared_symbol():
    header = open(os.path.join(ROOT, "include", "tmop_b200.h")).read()
    declared = set(re.findall(r"^(?:int|int64_t|const char \*|const double \*)\s*(tmop_\w+)\s*\(", header, re.M))
    assert declared, "no declarations parsed"
    assert declared == set(_lib.EXPORTED)
    lib = _lib.load()            # loads without a GPU; no compute calls here
    for name in declared:
        assert hasattr(lib, name), name


def test_no_cpu_fallback_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    mesh = P.build_box(2, (2, 2), 1)
    with pytest.raises(_lib.TmopLibraryError):
        P.TmopProblem(mesh, P.ObjectiveConfig(P.MetricId.MU_2, P.TargetSpec(P.TargetKind.IDEAL_UNIT)), 3)
    with pytest.raises(_lib.TmopLibraryError):
        P.metric_value(P.MetricId.MU_2, np.eye(2))


def test_product_does_not_import_oracle():
    pkg = os.path.join(ROOT, "paper_2205_12721_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith(".py"):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"^\s*(from|import)\s+oracle\b", src, re.M), f
                assert "tmop_oracle" not in src and "cpu_apply" not in src, f
