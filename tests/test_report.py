"""Reporting of the Kershaw benchmark driver (paper_2205_12721_b200/
kershaw_bench.py) against the reference's own outputs (bench.py:31-37,
244-330; fixture tests/golden/report_formats.npz written by the reference):
VTK Lagrange-hex point order, the VTK text of a Kershaw mesh, CSV header and
row formatting.  CPU only."""

import os

import numpy as np
import pytest

from conftest import load_golden

import paper_2205_12721_b200 as P
from paper_2205_12721_b200 import kershaw_bench as KB


@pytest.mark.parametrize("p", [1, 2, 3, 4])
def test_vtk_permutation_matches_reference(p):
    g = load_golden("report_formats")
    assert np.array_equal(KB.vtk_lagrange_hex_permutation(p), g[f"perm_p{p}"])


def test_vtk_text_matches_reference(tmp_path):
    g = load_golden("report_formats")
    mesh = P.apply_kershaw(P.build_cartesian(P.MeshSpec(3, 6, 2, 2, order=2)), 0.3, 0.3)
    path = os.path.join(tmp_path, "m.vtk")
    KB.write_vtk(mesh, path, title="kershaw initial mesh")
    assert open(path).read() == str(g["vtk_text"])


def test_csv_row_and_roundtrip_match_reference(tmp_path):
    g = load_golden("report_formats")
    times = {"total": 12.5, "gradient": 0.1 / 3, "hessian_setup": 1.0 / 7, "hessian_apply": 9.87654321,
             "linesearch": 2e-5, "objective": 0.01}
    rep = KB.RunReport(nx=24, ny=24, nz=24, order=1, n_quad=9, epsy=0.3, epsz=0.3, metric=303, preconditioned=True,
                       dofs_per_component=15625, dofs_total=46875, quad_points=24 ** 3 * 729, newton_iterations=13,
                       minres_iterations=650, times=times, f_initial=43335.601057054526, f_final=-4.279e-12,
                       relgrad_final=7.68e-10, min_det_initial=3.78e-06, min_det_final=4.6296296296296e-06,
                       max_dev_uniform=8.41e-9, status="failed", success=False)
    assert ",".join(KB.CSV_COLUMNS) == str(g["csv_header"])
    assert ",".join(rep.csv_row()) == str(g["csv_row"])
    path = os.path.join(tmp_path, "r.csv")
    KB.write_csv(rep, path)
    row = KB.read_csv_row(path)
    assert row["t_hess_apply_s"] == "9.8765432099999995" and row["status"] == "failed"
    text = KB.timing_breakdown(rep)
    assert "other" in text and "100.00%" in text


def test_bench_config_validation():
    with pytest.raises(ValueError):
        KB.BenchConfig(order=2, n_quad=2).validate()
    with pytest.raises(ValueError):
        KB.BenchConfig(limit_delta=-1.0).validate()
    with pytest.raises(Exception):
        KB.BenchConfig(nx=5).validate()        # Kershaw needs nx % 6 == 0 (mesh.py:50-60)
