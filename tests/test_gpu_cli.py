"""`cylspec` CLI end to end on the GPU: heat (manufactured and decay cases), poisson, ns and
transform write the reference's FieldFiles and manifest.json; results checked against the CPU
oracle (cylspec_main.cpp:67-282)."""
import json
import os
import subprocess
import tempfile

import numpy as np
import pytest

from tests.conftest import sample
from tests.inputs import rel_err

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_2206_04827_b200", "bin", "cylspec")


def run(*args):
    r = subprocess.run([BIN, *map(str, args)], capture_output=True, text=True, timeout=600,
                       cwd=tempfile.mkdtemp())  # never in the repo (failure_manifest.json lands under ./out)
    assert r.returncode == 0, r.stderr
    return r


def test_cli_heat_poisson_ns_transform(P, O, tmp_path):
    out = tmp_path / "heat"
    run("heat", "--m", 16, "--n", 16, "--p", 16, "--steps", 200, "--h", 0.01, "--out", out, "--output-every", 100)
    mf = json.loads((out / "manifest.json").read_text())
    assert mf["command"] == "heat" and abs(mf["final_time"] - 2.0) < 1e-12
    assert mf["max_rel_error"] < 1e-4
    # a number like the reference's (cylspec_main.cpp:108): the solver data's Sylvester residual
    assert isinstance(mf["worst_modal_residual"], float) and 0.0 < mf["worst_modal_residual"] < 1e-12
    assert [o["path"] for o in mf["outputs"]] == ["snapshot_0.ccf", "snapshot_1.ccf", "snapshot_2.ccf"]
    snap = P.read_field(out / "snapshot_2.ccf")
    assert snap.dtype == np.float64 and snap.shape == (16, 16, 16)

    out = tmp_path / "pois"
    run("poisson", "--m", 16, "--n", 16, "--p", 16, "--out", out)
    mf = json.loads((out / "manifest.json").read_text())
    assert mf["max_abs_error"] < 1e-8
    u = P.read_field(out / "solution.ccf")
    assert np.array_equal(P.read_field(out / "solution_values.ccf"), O.synthesize(u)) or \
        np.abs(P.read_field(out / "solution_values.ccf") - O.synthesize(u)).max() < 1e-12

    out = tmp_path / "ns"
    run("ns", "--m", 16, "--n", 16, "--p", 16, "--steps", 5, "--h", 1e-3, "--seed", 3, "--out", out)
    mf = json.loads((out / "manifest.json").read_text())
    assert abs(mf["final_time"] - 5e-3) < 1e-12 and np.isfinite(mf["final_divergence"])
    lam = P.read_field(out / "omega_toroidal.ccf")
    assert lam.dtype == np.complex128 and np.isfinite(lam).all()

    vals = O.synthesize(lam)
    P.write_field(tmp_path / "v.ccf", vals)
    out = tmp_path / "tr"
    run("transform", "--in", tmp_path / "v.ccf", "--out", out)
    assert rel_err(P.read_field(out / "coefficients.ccf"), O.analyze(vals)) < 1e-12


def test_cli_heat_decay_case(P, tmp_path):
    out = tmp_path / "d"
    run("heat", "--m", 16, "--n", 16, "--p", 16, "--steps", 20, "--case", "decay", "--seed", 5, "--out", out)
    mf = json.loads((out / "manifest.json").read_text())
    a0, a1 = P.read_field(out / "snapshot_0.ccf"), P.read_field(out / "snapshot_1.ccf")
    assert np.abs(a1).max() < np.abs(a0).max()  # pure diffusion decays
    assert "max_rel_error" not in mf
