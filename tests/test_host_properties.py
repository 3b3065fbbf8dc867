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
