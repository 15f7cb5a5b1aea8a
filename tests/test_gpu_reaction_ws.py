"""The warp-specialised fused reaction kernel (csrc/reaction_ws.cuh; d = 3, p = p_t in {2, 3}) against the
CPU oracle (reaction_mass's q = p+1 quadrature, assembly.py:287-347) and against reaction_tile, on
meshes that leave partial 2 x 4 x 2 element tiles in every direction, with the u0 lifting, on time-row
slabs and on a z slab (the sharded contexts)."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300)


def _spaces(nes, ne_t, p=3):
    import paper_2311_17500_b200 as mb
    from oracle.splines import make_space_time
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, n) for n in nes], mb.SplineSpace.uniform(p, ne_t))
    return st, make_space_time(3, p, nes, ne_t)


PS = pytest.mark.parametrize("p", [2, 3])


def _mr(op, x, kernel, store=0):
    """A x with the reaction evaluated by the given kernel (0 reaction_tile, 1 reaction_ws) in the fused
    (store 0) or the stored-coefficient mode (store 1)."""
    from paper_2311_17500_b200 import _lib
    _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
    _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, kernel)
    return op.matvec(x)


@pytest.mark.parametrize("p", [2, 3])
@pytest.mark.parametrize("nes,ne_t", [((5, 7, 3), 6), ((2, 4, 2), 4), ((1, 1, 1), 1), ((9, 3, 5), 3)])
def test_reaction_ws_matches_oracle_and_tile_kernel(nes, ne_t, p):
    import paper_2311_17500_b200 as mb
    from oracle import assembly as oasm
    st, ost = _spaces(nes, ne_t, p)
    T, D = 1.3, 2e-2
    rng = np.random.default_rng(sum(nes) + ne_t)
    N = st.num_dof
    u, w, x = rng.uniform(0, 1, N), rng.uniform(0, 0.1, N), rng.uniform(-1, 1, N)
    op = mb.KroneckerOperator(st, T, 1.0, D, RM, u=u, w=w)
    op0 = mb.KroneckerOperator(st, T, 1.0, D, {"c1": 0.0, "a": 0.0, "c2": 0.0})     # Galerkin part alone
    y0 = op0.matvec(x)
    y_ws = _mr(op, x, 1) - y0
    y_tile = _mr(op, x, 0) - y0
    y_ref = oasm.reaction_matvec(ost, T, RM, u, w, x)
    assert rel(y_ws, y_ref) < 1e-12
    assert rel(y_tile, y_ref) < 1e-12
    assert rel(y_ws, y_tile) < 1e-13
    # the stored-coefficient mode of both kernels (c_w written once by the kernel's own RX_PRE pass)
    for kernel in (0, 1):
        y_st = _mr(op, x, kernel, store=1) - y0
        assert rel(y_st, y_ref) < 1e-12
        assert rel(_mr(op, x, kernel, store=1) - y0, y_st) == 0.0      # a second apply reuses c_w
    # repeated applies are bitwise identical (one writer per entry per colour launch)
    assert np.array_equal(_mr(op, x, 1), _mr(op, x, 1))


@PS
def test_reaction_ws_with_lift_matches_tile_kernel(p):
    """The lifted slab (row -1) of u and of x (mi_op_apply_lift) enters through the producers' copies."""
    import paper_2311_17500_b200 as mb
    st, _ = _spaces((5, 6, 3), 5, p)
    rng = np.random.default_rng(3)
    N, ns = st.num_dof, st.num_space
    u, w, x = rng.uniform(0, 1, N), rng.uniform(0, 0.1, N), rng.uniform(-1, 1, N)
    lift = rng.uniform(0, 1, ns)
    op = mb.KroneckerOperator(st, 0.9, 1.0, 1e-2, RM, u=u, w=w, lift=lift)
    from paper_2311_17500_b200 import _lib
    out = {}
    for store in (0, 1):
        _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
        for kernel in (0, 1):
            _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, kernel)
            out[store, kernel] = (op.matvec(x), op.lift_apply().cpu().numpy())
    for key in ((0, 1), (1, 0), (1, 1)):
        assert rel(out[key][0], out[0, 0][0]) < 1e-13
        assert rel(out[key][1], out[0, 0][1]) < 1e-13


@PS
def test_reaction_ws_on_time_row_slabs(p):
    """Time-row slabs (KroneckerOperator(time_rows=...)): rows outside the slab are zero slabs."""
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import _lib
    st, _ = _spaces((4, 5, 3), 9, p)
    rng = np.random.default_rng(5)
    N, ns, nt = st.num_dof, st.num_space, st.num_time
    u, w, x = rng.uniform(0, 1, N), rng.uniform(0, 0.1, N), rng.uniform(-1, 1, N)
    r0, r1 = 3, 8
    sl = slice(r0 * ns, r1 * ns)
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-2, RM, u=u[sl], w=w[sl], time_rows=(r0, r1))
    ys = []
    for store in (0, 1):
        _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
        for kernel in (0, 1):
            _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, kernel)
            ys.append(op.matvec(x[sl]))
    for y in ys[1:]:
        assert rel(y, ys[0]) < 1e-13


@PS
def test_reaction_ws_on_z_slab(p):
    """The z-slab operator of the space-sharded solve: the reaction runs on the input slab (owned planes
    + halos) and only the owned planes are kept."""
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import _lib
    st, _ = _spaces((4, 4, 9), 4, p)
    rng = np.random.default_rng(8)
    n1, n2, n3 = (s.dimension for s in st.spatial)
    nt = st.num_time
    z_lo, z_hi = 4, 8
    h_lo, h_hi = min(p, z_lo), min(p, n3 - z_hi)
    nin = (z_hi + h_hi - (z_lo - h_lo)) * n1 * n2
    u, w, x = (rng.uniform(0, 1, nt * nin), rng.uniform(0, 0.1, nt * nin), rng.uniform(-1, 1, nt * nin))
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-2, RM, u=u, w=w, z_planes=(z_lo, z_hi))
    ys = []
    for store in (0, 1):
        _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
        for kernel in (0, 1):
            _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, kernel)
            ys.append(op.matvec(x))
    for y in ys[1:]:
        assert rel(y, ys[0]) < 1e-13


def test_reaction_kernel_selector_rejects_unsupported_shapes():
    import paper_2311_17500_b200 as mb
    from paper_2311_17500_b200 import _lib
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 3) for _ in range(2)], mb.SplineSpace.uniform(2, 3))
    op = mb.KroneckerOperator(st, 1.0, 1.0, 1e-2, RM)
    with pytest.raises(Exception):
        _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, 1)
    _lib.call("mi_op_set_reaction_kernel", op.ctx.handle, 0)
