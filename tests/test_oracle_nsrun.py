"""Oracle NSStepper::seed and ns_run (proj/src/ptns.cpp:195-203, 269-324). test_ptns.cpp is a placeholder, so
the pins are the code's own semantics: a stepper seeded with a run's history continues that run bit for bit,
the substeps bootstrap equals its hand-built restatement from the public pieces, and both bootstraps converge
to the same trajectory as h -> 0 (the substeps start is the more accurate one: BDF2 at h/32 vs BDF1 at h)."""
import numpy as np
import pytest

from tests.inputs import hermitian_coeffs, rel_err

M = N = P_ = 8


def _init(scale=0.05):
    return hermitian_coeffs(M, N, P_, 0.6, 11) * scale, hermitian_coeffs(M, N, P_, 0.6, 12) * scale


def _history(O, lam, gam, re, h, k):
    """omega history (newest first) and nonlinear history of a ramp run after k steps."""
    st = O.NSStepper(lam, gam, re, h)
    oh = [(O.parity_project(lam, 0), O.parity_project(gam, 0))]
    for _ in range(k):
        st.step()
        oh.insert(0, st.omega())
    nh = [O.nonlinear(*O.velocity_from_vorticity(*w), *w) for w in oh[1:]]
    return st, oh, nh


def test_seed_continues_a_run_bit_for_bit(O):
    lam, gam = _init()
    run, oh, nh = _history(O, lam, gam, 100.0, 1e-3, 3)
    seeded = O.NSStepper(*oh[0], 100.0, 1e-3)
    seeded.seed(oh, nh, 3e-3, 3)
    run.step(2)
    seeded.step(2)
    (l, g), (rl, rg) = seeded.omega(), run.omega()
    assert np.array_equal(l, rl) and np.array_equal(g, rg)
    assert seeded.steps_taken == 5 and abs(seeded.time - 5e-3) < 1e-15


def test_seed_errors(O):
    lam, gam = _init()
    st = O.NSStepper(lam, gam, 100.0, 1e-3)
    with pytest.raises(O.OracleError, match="empty history"):
        st.seed([], [], 0.0, 0)
    st.seed([(lam, gam)], [], 3e-3, 3)  # order 4 from one entry: bdf_rhs refuses (timestep.cpp:41-42)
    with pytest.raises(O.OracleError, match="insufficient history"):
        st.step()


def test_ns_run_ramp_equals_stepper(O):
    lam, gam = _init()
    l, g, t = O.ns_run(lam, gam, 5, 100.0, 1e-3)
    st = O.NSStepper(lam, gam, 100.0, 1e-3)
    st.step(5)
    rl, rg = st.omega()
    assert np.array_equal(l, rl) and np.array_equal(g, rg) and abs(t - 5e-3) < 1e-15


@pytest.mark.parametrize("order", [2, 3])
def test_ns_run_substeps_equals_hand_built(O, order):
    lam, gam = _init()
    re, h, steps = 100.0, 2e-3, order + 1
    l, g, t = O.ns_run(lam, gam, steps, re, h, order=order, bootstrap="substeps")
    fine = O.NSStepper(lam, gam, re, h / 32, order=2)
    hist = [(lam, gam)]
    for _ in range(order - 1):
        fine.step(32)
        hist.insert(0, fine.omega())
    replay = [O.nonlinear(*O.velocity_from_vorticity(*w), *w) for w in hist[1:]]
    st = O.NSStepper(*hist[0], re, h, order=order)
    st.seed(hist, replay, (order - 1) * h, order - 1)
    st.step(steps - (order - 1))
    rl, rg = st.omega()
    assert np.array_equal(l, rl) and np.array_equal(g, rg) and abs(t - steps * h) < 1e-15


def test_ns_run_substeps_order1_and_zero_steps_are_the_ramp(O):
    lam, gam = _init()
    a = O.ns_run(lam, gam, 2, 100.0, 1e-3, order=1, bootstrap="substeps")
    b = O.ns_run(lam, gam, 2, 100.0, 1e-3, order=1)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    z = O.ns_run(lam, gam, 0, 100.0, 1e-3, bootstrap="substeps")
    assert np.array_equal(z[0], O.parity_project(lam, 0)) and z[2] == 0.0


def test_bootstraps_agree_to_the_ramp_start_error(O):
    # both integrate the same equation to the same final time: they differ by the ramp's BDF1 / BDF2 start
    # error, and the gap shrinks as h does
    lam, gam = _init(0.2)
    gaps = []
    for h, steps in ((4e-3, 4), (2e-3, 8)):
        a = O.ns_run(lam, gam, steps, 50.0, h, order=3, bootstrap="substeps")
        b = O.ns_run(lam, gam, steps, 50.0, h, order=3)
        gaps.append(max(rel_err(a[0], b[0]), rel_err(a[1], b[1])))
    assert 0 < gaps[1] < gaps[0] < 5e-2 and gaps[0] / gaps[1] > 2.5
