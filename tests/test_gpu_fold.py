"""GPU: the even/odd (folded) spatial transforms of P^-1 (csrc/mode_fold.cuh)
against the dense n x n mode products on the same eigenbasis.

Uniform open knot vectors give centrosymmetric univariate pencils, so
factors.spatial_eigs returns an exactly mirrored basis and the device applies
U_l^T / U_l as two half-size products.  P^-1 is the same operator either way:
the two paths agree to 1e-13 relative (the reference-facing P^-1 parity is
tests/test_gpu_parity.py, which now runs the folded path).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _pc(st, fold):
    import paper_2311_17500_b200 as mb
    old = os.environ.pop("MI_NO_FOLD", None)
    if not fold:
        os.environ["MI_NO_FOLD"] = "1"
    try:
        return mb.FastDiagPreconditioner.build(st, 1.0, 1.0, [1e-3, 4e-4, 4e-4][:st.num_spatial_dims],
                                               0.13 * 0.26)
    finally:
        os.environ.pop("MI_NO_FOLD", None)
        if old is not None:
            os.environ["MI_NO_FOLD"] = old


# (d, p, ne, ne_t): n = ne + p spatial functions (ne may differ per direction); hs = n - n // 2
# covers every instantiated half size (1, 2, 3, 5, 7 tiles of 8), odd and even n, one size past
# the folded range (dense fallback), contiguous-mode tiles with an odd element count (n odd, odd
# row count in the last tile), and strided modes whose HBM parity flips at a slab boundary (n even,
# inner extent odd)
SHAPES = [(1, 2, 30, 10), (2, 3, 40, 6), (3, 1, 6, 4), (3, 2, 13, 6), (3, 3, 20, 8), (3, 2, 64, 4),
          (3, 3, 96, 2), (2, 2, 120, 4), (1, 2, 31, 4), (2, 2, 11, 4), (2, 3, (20, 13), 5),
          (3, 2, (11, 14, 9), 3)]


@pytest.mark.parametrize("shape", SHAPES)
def test_folded_transforms_match_dense(shape):
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import _lib
    d, p, ne, ne_t = shape
    ne = (ne,) * d if np.isscalar(ne) else ne
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, e) for e in ne], mb.SplineSpace.uniform(p, ne_t))
    Pf, Pd = _pc(st, True), _pc(st, False)
    for l in range(d):
        n = ne[l] + p
        hs = n - n // 2
        assert _lib.load().mi_pc_fold(Pf.ctx.handle, l) == hs   # past 56 the launch falls back to dense
        assert _lib.load().mi_pc_fold(Pd.ctx.handle, l) == 0
    r = np.random.default_rng(3).uniform(-1, 1, Pf.shape[0])
    zf, zd = Pf.apply(r), Pd.apply(r)
    err = np.linalg.norm(zf - zd) / np.linalg.norm(zd)
    assert err < 1e-13, err


def test_nonuniform_knots_use_dense_path():
    """A graded knot vector breaks the mirror symmetry: no fold, dense products."""
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import _lib
    p = 2
    inner = np.linspace(0, 1, 12)[1:-1] ** 1.5
    knots = np.concatenate([[0.0] * (p + 1), inner, [1.0] * (p + 1)])
    sp = mb.SplineSpace(knots, p)
    st = mb.SpaceTimeSpace([sp, sp], mb.SplineSpace.uniform(p, 6))
    P = _pc(st, True)
    assert _lib.load().mi_pc_fold(P.ctx.handle, 0) == 0
