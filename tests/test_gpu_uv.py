"""UPDATE_VELOCITY with a zero upwind blend (the reference default, alpha = 0):
the device evaluates the blend terms only for zero fluxes (sf_uv.cuh), which
must stay bitwise the reference's f + alpha * X -- including signed zeros,
which the FNV checksum hashes (bench.hpp:24-39)."""
import numpy as np
import pytest

from oracle.oracle import Case, Oracle
from test_gpu_parity import dev_from_case, same

pytestmark = pytest.mark.gpu


def _zero_heavy(shape, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1.0, 1.0, size=shape)
    pick = rng.random(shape)
    a[pick < 0.35] = 0.0
    a[(pick >= 0.35) & (pick < 0.6)] = -0.0
    a[(pick >= 0.6) & (pick < 0.7)] = 0.5  # equal neighbours: differences are +0
    return a


@pytest.mark.parametrize("blend", [0.0, -0.0, 0.25])
@pytest.mark.parametrize("seed", [1, 2])
def test_update_velocity_zero_blend_keeps_signed_zeros_bitwise(ref_available, blend, seed):
    c = Case(extents=(37, 21, 13), symmetry_z=False, lid_speed=0.0, blend=blend, viscosity=0.0125)
    o = Oracle(c, "ref")
    d = dev_from_case(c)
    shape = (13, 21, 37)
    for k, f in enumerate(("vx", "vy", "vz", "p")):
        a = _zero_heavy(shape, 10 * seed + k)
        o.scatter(f, a)
        d.scatter(f, a)
    o.invalidate_all_ghosts()
    d.invalidate_all_ghosts()
    o.provisional(0.0078125)
    d.provisional(0.0078125)
    for f in ("vx", "vy", "vz"):
        g, w = d.gather(f), o.gather(f)
        assert same(g, w), (f, int(np.sum(g.view(np.uint64) != w.view(np.uint64))))
    zeros = [int(np.sum(o.gather(f) == 0.0)) for f in ("vx", "vy", "vz")]
    assert min(zeros) > 0, zeros  # the zero-flux cases were exercised
