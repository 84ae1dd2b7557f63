"""Pins of oracle/mmoc.py (MMOC): zero velocity returns the nodal values; constants are
transported unchanged; on the flat shell a linear velocity u = A x is interpolated exactly, RK4 on the
linear ODE X' = -A X is its 4th-order Taylor polynomial, so for linear T the result is exactly
c . P4(-tau A) x (brute-force closed form) for nodes whose paths stay inside the polyhedral shell."""
import numpy as np
import pytest

from oracle.mmoc import mmoc
from oracle.operators import node_coords
from oracle.refine import build_level
from workload import icoshell, uniform_from_keys, uniform_vec


@pytest.fixture(scope="module")
def shell_l1():
    m = icoshell(3, 2)
    return build_level(m.verts, m.tets, m.vtag, 1)


def test_zero_velocity_and_constants(shell_l1):
    lm = shell_l1
    T = uniform_from_keys(lm.p2_keys, 3, 0)
    z = np.zeros(3 * lm.n_p2)
    nodes = np.arange(0, lm.n_p2, 7)
    assert np.abs(mmoc(lm, True, T, z, z, 0.05, nodes) - T[nodes]).max() < 1e-13
    u = 0.3 * uniform_vec(lm.p2_keys, 2)
    one = np.ones(lm.n_p2)
    assert np.abs(mmoc(lm, True, one, u, 0.5 * u, 0.05, nodes) - 1.0).max() < 1e-13


def test_linear_velocity_rk4_closed_form():
    m = icoshell(3, 2)
    lm = build_level(m.verts, m.tets, m.vtag, 1)
    w, tau = 2.0, 0.1
    A = np.array([[0.0, -w, 0.3], [w, 0.0, -0.2], [-0.3, 0.2, 0.0]])   # skew: |x| preserved by the flow
    x = lm.p2_xt
    u = (x @ A.T).ravel()
    c = np.array([0.4, -0.9, 1.3])
    T = x @ c
    r = np.linalg.norm(x, axis=1)
    nodes = np.nonzero((r > 0.62) & (r < 0.8))[0]
    Z = -tau * A
    P4 = np.eye(3) + Z + Z @ Z / 2 + Z @ Z @ Z / 6 + Z @ Z @ Z @ Z / 24
    exact = (x[nodes] @ P4.T) @ c
    got = mmoc(lm, False, T, u, u, tau, nodes)
    assert len(nodes) > 50 and np.abs(got - exact).max() < 1e-13
    # time interpolation: u_old = 0 halves the velocity at the midpoint stages -> different result
    got2 = mmoc(lm, False, T, u, np.zeros_like(u), tau, nodes)
    assert np.abs(got2 - exact).max() > 1e-4
