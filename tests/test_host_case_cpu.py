"""CPU: the product's host half of case loading (grid, bodies, M, L, G, boundary couplings) is
bit-identical to the reference's (config.hpp, grid.hpp, body.hpp, operators.hpp:75-228)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_1109_3524_b200 import ibm
from tests import helpers as H

CASES = [("cavity", 0.0), ("cylinder_re40_smoke", 0.0), ("flapping_smoke", 0.0), ("cylinder_re40", 0.0),
         ("cylinder_re3000", 0.0), ("flapping", 0.0), ("uniform_cylinder", 30.72 / 256)]


@pytest.mark.parametrize("name,h_min", CASES)
def test_host_case_matches_reference(ref, name, h_min):
    hc = ibm.HostCase(H.case(name), h_min=h_min)
    rc = ref.case(H.case(name), h_min)
    assert (hc.nx, hc.ny, hc.n_q, hc.n_p, hc.n_b, hc.n_lambda) == (rc.nx, rc.ny, rc.n_q, rc.n_p, rc.n_b,
                                                                    rc.n_lambda)
    g = rc.grid()
    for k in O.RefCase.GRID:
        assert np.array_equal(hc.array(k), g[k]), k
    assert np.array_equal(hc.array("uniform"), g["uniform"])
    bd = rc.bodies()
    for k in ("x", "y", "ub_x", "ub_y", "ds"):
        assert np.array_equal(hc.array("body_" + k), bd[k]), k
    for k in ("L", "G"):
        rows, cols, rp, ci, v = hc.csr(k)
        H.assert_csr_equal(O.Csr(rows, cols, rp, ci, v), rc.op(k))
    assert np.array_equal(hc.array("visc_bc"), rc.visc_bc())
    assert np.array_equal(hc.array("boundary"), rc.boundary())


def test_moving_body_kinematics_match_reference(ref):
    """LagrangianBody::move_to along a flapping trajectory (body.hpp:63-148)."""
    hc = ibm.HostCase(H.case("flapping_smoke"))
    rc = ref.case(H.case("flapping_smoke"))
    for _ in range(3):
        rc.step()
        hc.move(rc.time())
        bd = rc.bodies()
        for k in ("x", "y", "ub_x", "ub_y"):
            assert np.array_equal(hc.array("body_" + k), bd[k]), k


def test_config_errors():
    import os
    import tempfile
    bad = "[grid]\ndomain = 0 1 0 1\nuniform = 0 1 0 1\nh_min = 0.1\nratio = 1 1 1 1\n[fluid]\nre = 10\n" \
          "[time]\ndt = 0.1\nn_steps = 1\n[bogus]\n"
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as f:
        f.write(bad)
    try:
        with pytest.raises(ValueError, match="unknown section"):
            ibm.HostCase(f.name)
    finally:
        os.unlink(f.name)
    with pytest.raises(ValueError, match="cannot open"):
        ibm.HostCase("/nonexistent.cfg")
