"""Host-side helpers of the drop-in API (no GPU): the reference's
test_prescribed_motion_is_second_order (pkg/tests/test_hydro.py:263-276) on
paper_2112_07075_b200.hydro.advance_positions."""

import numpy as np


def test_prescribed_motion_is_second_order():
    from paper_2112_07075_b200.hydro import advance_positions

    # dx/dt = x has the exact solution x0 * exp(t); midpoint stepping must show global
    # error O(dt^2): slope 2 over dt halvings
    x0 = np.linspace(0.5, 1.5, 7).reshape(-1, 1)
    errs = []
    for nsteps in (8, 16, 32, 64):
        dt = 1.0 / nsteps
        x = x0.copy()
        for _ in range(nsteps):
            x = advance_positions(x, dt, lambda y, t: y)
        errs.append(np.abs(x - x0 * np.e).max())
    slopes = np.log2(np.array(errs[:-1]) / np.array(errs[1:]))
    assert np.all(np.abs(slopes - 2.0) < 0.1)


def test_tmop_host_metrics_fd_consistent():
    """The host evaluators of the TMOP metrics (paper_2112_07075_b200.meshopt, the closed
    forms the device kernels use): dmu matches central differences of mu (SPEC: 1e-6) and
    the directional second derivative matches differences of dmu (1e-5)."""
    from paper_2112_07075_b200 import meshopt

    rng = np.random.default_rng(3)
    for d, m in [(2, meshopt.metric_for(2)), (3, meshopt.metric_for(3)), (2, meshopt.metric_for(2, True)),
                 (3, meshopt.metric_for(3, True))]:
        T = np.eye(d)[None] + 0.2 * rng.standard_normal((6, d, d))
        dT = rng.standard_normal((6, d, d))
        h = 1e-6
        fd = (m.mu(T + h * dT) - m.mu(T - h * dT)) / (2 * h)
        an = np.einsum("nij,nij->n", m.dmu(T), dT)
        assert np.max(np.abs(fd - an)) <= 1e-6 * np.max(np.abs(an))
        fd2 = (m.dmu(T + h * dT) - m.dmu(T - h * dT)) / (2 * h)
        an2 = np.einsum("nmzkl,nkl->nmz", m.d2mu(T), dT)
        assert np.max(np.abs(fd2 - an2)) <= 1e-5 * np.max(np.abs(an2))
        assert np.allclose(m.mu(np.eye(d)[None]), 0.0, atol=1e-15)
