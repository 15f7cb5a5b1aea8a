"""GPU: the fused FD time stage (csrc/tstage.cuh: Q^T, arrowhead, Q in one kernel per
column tile) at every instantiated row-block count, against the reference-pinned
oracle P^-1 (oracle/fastdiag.py, complex pencil as linalg.py:317-353).

nt = ne_t + p - 1 constrained time functions; the kernel instance is the smallest
MB in {4, 8, 13, 17, 25, 33, 41, 49} with 8 MB >= nt (25 is the cfg-4 bench size,
nt = 194).  The 2D cases give several column tiles plus a partial last tile.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}

# (d, ne, ne_t) at p = 2
CASES = [(1, 10, 30), (1, 10, 60), (2, 13, 100), (1, 10, 130), (2, 13, 193), (1, 10, 250), (1, 10, 320),
         (1, 10, 380)]


@pytest.mark.parametrize("case", CASES)
def test_time_stage_matches_oracle(case):
    import paper_2311_17500_b200 as mb
    from oracle import problem as oprob
    from oracle.splines import make_space_time
    d, ne, ne_t = case
    p = 2
    ost = make_space_time(d, p, ne, ne_t)
    opc = oprob.preconditioner(ost, 1.0, 1.0, 1e-3, RM)
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, ne) for _ in range(d)], mb.SplineSpace.uniform(p, ne_t))
    P = mb.FastDiagPreconditioner.build(st, 1.0, 1.0, 1e-3, RM["a"] * RM["c1"])
    r = np.random.default_rng(7).uniform(-1, 1, P.shape[0])
    z, zr = P.apply(r), opc.apply(r)
    err = np.linalg.norm(z - zr) / np.linalg.norm(zr)
    assert err < 1e-12, err
