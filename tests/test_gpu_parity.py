"""GPU parity: the CUDA path (through the C ABI) vs the reference-pinned oracle
and the reference's own golden vectors.

Tolerances (fp64): component applies <= 1e-12 relative; GMRES iteration
counts equal and solutions <= 1e-10 relative (north_star parity bar).
"""

import numpy as np
import pytest

from cases import CASES, load, oracle_objects

pytestmark = pytest.mark.gpu

RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


def product_objects(g, with_su=True, u=None, w=None):
    import paper_2311_17500_b200 as mb
    p = int(g["p"])
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(p, int(n)) for n in g["ne"]],
                           mb.SplineSpace.uniform(p, int(g["ne_t"])))
    sig = np.atleast_1d(g["sigma"])
    sig = float(sig[0]) if sig.size == 1 else sig
    stab = mb.Stabilization(st, g["theta"], float(g["su_tol"]), 1.0) if with_su else None
    op = mb.KroneckerOperator(st, float(g["T"]), 1.0, sig, RM, u=u, w=w, stabilization=stab)
    P = mb.FastDiagPreconditioner.build(st, float(g["T"]), 1.0, sig, 0.13 * 0.26, context=op.ctx)
    return st, op, P


@pytest.mark.parametrize("name", CASES)
def test_separable_operator(name):
    g = load(name)
    _, op, _ = product_objects(g, with_su=False)
    assert rel(op.matvec(g["x"]), g["y_sep"]) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_full_operator_zero_iterate(name):
    g = load(name)
    _, op, _ = product_objects(g)
    assert rel(op.matvec(g["x"]), g["y_a"]) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_preconditioner(name):
    g = load(name)
    _, op, P = product_objects(g)
    assert rel(P.apply(g["x"]), g["z_pc"]) < 1e-12
    assert rel(P.apply(op.matvec(g["x"])), g["z_pc_ya"]) < 1e-12


@pytest.mark.parametrize("name", CASES)
def test_gmres_matches_reference(name):
    import paper_2311_17500_b200 as mb
    g = load(name)
    _, op, P = product_objects(g)
    x, it, hist = mb.gmres(op, g["rhs"], precond=P, tol=1e-8, max_iter=400)
    assert it == int(g["gm_a_it"])
    assert rel(x, g["gm_a_x"]) < 1e-10
    np.testing.assert_allclose(hist, g["gm_a_hist"], rtol=1e-6, atol=1e-14)


def test_dimension_mismatch_and_torch_inputs():
    import torch
    g = load("case_2d_p2")
    _, op, P = product_objects(g)
    with pytest.raises(ValueError, match="dimension mismatch"):
        op.matvec(np.zeros(op.shape[0] + 1))
    with pytest.raises(ValueError, match="dimension mismatch"):
        P.apply(np.zeros(3))
    xt = torch.from_numpy(g["x"]).cuda()
    yt = op.matvec(xt)
    assert yt.is_cuda and rel(yt.cpu().numpy(), g["y_a"]) < 1e-12


def test_gmres_known_answers_device():
    """tests/test_linalg.py:177-214 semantics on the device path."""
    import paper_2311_17500_b200 as mb
    g = load("case_2d_p2")
    _, op, P = product_objects(g)
    x, it, hist = mb.gmres(op, np.zeros(op.shape[0]), precond=P)
    assert it == 0 and hist == [0.0] and not np.any(x)
    with pytest.raises(mb.NonConvergenceError) as e:
        mb.gmres(op, g["rhs"], precond=P, tol=1e-14, max_iter=3)
    assert e.value.iterations == 3 and len(e.value.residuals) == 4


@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("store", [0, 1])
def test_operator_general_iterate_reaction(name, store):
    """Variant B: M_R (q=p+1 Gauss, Rogers-McCulloch linearisation) at u, w != 0, with C_r formed
    in every apply (store 0) and stored once per operator build (store 1)."""
    from paper_2311_17500_b200 import _lib
    g = load(name)
    _, op, _ = product_objects(g, u=g["u"], w=g["w"])
    assert not op.zero_iterate
    _lib.call("mi_op_set_reaction_store", op.ctx.handle, store)
    assert rel(op.matvec(g["x"]), g["y_b"]) < 1e-12
    assert rel(op.matvec(g["x"]), g["y_b"]) < 1e-12         # a second apply reuses the stored c_w
    # the reaction part alone: A_b x - (A_a x - a c1 M_t M_s x) = M_R x
    _, op_sep, _ = product_objects(g, with_su=False, u=g["u"], w=g["w"])
    _, op_sep0, _ = product_objects(g, with_su=False)
    y_mr = op_sep.matvec(g["x"]) - op_sep0.matvec(g["x"])
    y_ref = g["y_mr"] - (g["y_sep"] - op_sep0_galerkin(g))
    assert rel(y_mr, y_ref) < 1e-10


def op_sep0_galerkin(g):
    """Galerkin part without reaction, from the oracle (test helper)."""
    from oracle import problem
    from cases import space_of, sigma_of
    st = space_of(g)
    op = problem.operator_terms(st, float(g["T"]), 1.0, sigma_of(g), {"c1": 0.0, "a": 0.0, "c2": 0.0})
    return op.matvec(g["x"])


@pytest.mark.parametrize("name", CASES)
def test_gmres_general_iterate_matches_reference(name):
    import paper_2311_17500_b200 as mb
    g = load(name)
    _, op, P = product_objects(g, u=g["u"], w=g["w"])
    x, it, hist = mb.gmres(op, g["rhs"], precond=P, tol=1e-8, max_iter=400)
    assert it == int(g["gm_b_it"])
    assert rel(x, g["gm_b_x"]) < 1e-10


@pytest.mark.parametrize("depth", [1, 2])
def test_apply_stream_matches_serial(depth):
    """ApplyStream (copy-in / apply / copy-out on three streams) is bitwise the serial path."""
    import torch
    import paper_2311_17500_b200 as mb
    g = load("case_3d_p3")
    _, op, P = product_objects(g)
    n = op.shape[0]
    rng = np.random.default_rng(7)
    xs = [torch.from_numpy(rng.uniform(-1, 1, n)).pin_memory() for _ in range(5)]
    zs = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(5)]
    ys = [torch.empty(n, dtype=torch.float64).pin_memory() for _ in range(5)]
    mb.ApplyStream(op, P, depth=depth).run(xs, zs)
    mb.ApplyStream(op, None, depth=depth).run(xs, ys)
    torch.cuda.synchronize()
    for x, z, y in zip(xs, zs, ys):
        ref_y = op.matvec(x.numpy())
        ref_z = P.apply(ref_y)
        assert np.array_equal(y.numpy(), ref_y)
        assert np.array_equal(z.numpy(), ref_z)
    with pytest.raises(ValueError):
        mb.ApplyStream(op, P).run(xs[:1], [torch.empty(3, dtype=torch.float64)])


@pytest.mark.parametrize("k", [1, 5, 13, 31, 40])
def test_fused_cgs_passes_are_bitwise_the_two_pass_kernels(k):
    """mi_cgs_pass / mi_cgs_norm_pass (one read of V per CGS2 subtraction + reduction) equal
    mi_sub_combination followed by mi_dots bit for bit (linalg.py:405-412)."""
    import torch
    from paper_2311_17500_b200.device import DeviceContext
    from paper_2311_17500_b200.krylov import DeviceVecOps
    import paper_2311_17500_b200 as mb
    st = mb.SpaceTimeSpace([mb.SplineSpace.uniform(2, 30)], mb.SplineSpace.uniform(2, 40))
    ctx = DeviceContext(st, 0)
    ops = DeviceVecOps(ctx)
    n = 1_000_003
    g = torch.Generator(device="cuda").manual_seed(k)
    V = torch.randn(k + 1, n, dtype=torch.float64, device="cuda", generator=g)
    w0 = torch.randn(n, dtype=torch.float64, device="cuda", generator=g)
    h = torch.randn(k, dtype=torch.float64, device="cuda", generator=g)
    wa, wb = w0.clone(), w0.clone()
    ha, hb = torch.zeros(k, dtype=torch.float64, device="cuda"), torch.zeros(k, dtype=torch.float64, device="cuda")
    ops.sub_comb(V, k, h, wa)
    ops.dots(V, k, wa, ha)
    ops.sub_dots(V, k, h, wb, hb)
    assert torch.equal(wa, wb) and torch.equal(ha, hb)
    na, nb = torch.zeros(1, dtype=torch.float64, device="cuda"), torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.sub_comb(V, k, ha, wa)
    ops.dots(wa.view(1, -1), 1, wa, na)
    ops.sub_norm(V, k, hb, wb, nb)
    assert torch.equal(wa, wb) and torch.equal(na, nb)
    ctx.close()


@pytest.mark.parametrize("name", ["case_3d_p3", "case_3d_p2_front", "case_2d_p2"])
@pytest.mark.parametrize("nparts", [1, 2, 3])
def test_matvec_from_host_is_bitwise_matvec(name, nparts):
    """KroneckerOperator.matvec_from_host (H2D in z-plane chunks under the stencil of the chunks already
    copied, mi_op_apply_from_host) == matvec of the device vector, bit for bit, with and without M_R."""
    import torch
    g = load(name)
    for u, w in ((None, None), (g["u"], g["w"])):
        _, op, _ = product_objects(g, u=u, w=w)
        xh = torch.from_numpy(g["x"]).pin_memory()
        y = op.matvec_from_host(xh, nparts=nparts)
        ref = op.matvec(xh.cuda())
        assert torch.equal(y, ref)
        assert rel(y.cpu().numpy(), g["y_a"] if u is None else g["y_b"]) < 1e-12
