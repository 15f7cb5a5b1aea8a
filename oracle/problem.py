"""Term list of the potential system and the seeded benchmark inputs.

Restates ``_Workspace.operator`` (solver.py:213-236) and the CPU-baseline
construction of SURVEY.md Appendix C / section 8(d).
TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""

import numpy as np

from . import assembly as asm
from . import stab
from .fastdiag import FastDiag
from .splines import make_space_time

RM = dict(a=0.13, c1=0.26, c2=0.1, b=0.013, d_e=1.0)

# BASELINE.json configs: (d, p, n_el space, n_el time, sigma)
CONFIGS = {
    1: dict(d=1, p=2, ne=64, ne_t=64, sigma=(1e-3,)),
    2: dict(d=2, p=3, ne=128, ne_t=256, sigma=(1e-3, 1e-3)),
    3: dict(d=3, p=2, ne=64, ne_t=128, sigma=(1e-3, 4e-4, 4e-4)),
    4: dict(d=3, p=3, ne=96, ne_t=192, sigma=(1e-3, 1e-3, 1e-3)),
}


def front_indicator(st):
    """SURVEY 8(d) seeded SU indicator (deterministic, no RNG).

    Theta[i_t, i_s] = clip(exp(-((g1(i_s) - 0.2 - 0.5 g_t(i_t)) / 0.08)^2), 0, 1)
    with g1 the direction-1 Greville abscissa of i_s, g_t the constrained
    time Greville abscissa.
    """
    g1 = st.spatial[0].greville()
    n1 = g1.size
    gs = np.tile(g1, st.num_space // n1)
    gt = st.time_greville()
    th = np.exp(-(((gs[None, :] - 0.2 - 0.5 * gt[:, None]) / 0.08) ** 2))
    return np.clip(th, 0.0, 1.0)


def operator_terms(st, T, cm, sigma, consts, u=None, w=None, su_terms=(), lengths=None):
    """solver.py:213-236 term list (+ anisotropic K_sigma).

    Returns a KronOp.  ``sigma`` is a scalar D or one conductivity per
    direction.  With u = w = 0 (or None) the reaction is the Kronecker term
    c1*a M_t x M_s; otherwise the q=p+1 reaction mass is a CSR correction.
    """
    Wt, Mt = asm.time_factors(st, T)
    sig = np.atleast_1d(np.asarray(sigma, float))
    if sig.size == 1:
        Ms, Ks = asm.box_spatial(st.spatial, lengths)
        terms = [(cm, Wt, Ms), (float(sig[0]), Mt, Ks)]
    else:
        Ms, Ks = asm.box_spatial(st.spatial, lengths, diffusion=sig)
        terms = [(cm, Wt, Ms), (1.0, Mt, Ks)]
    corr = None
    zero = (u is None or not np.any(u)) and (w is None or not np.any(w))
    if zero:
        terms.append((consts["c1"] * consts["a"], Mt, Ms))
    else:
        corr = asm.reaction_mass(st, T, consts, u, w, lengths)
    terms.extend(su_terms)
    return asm.KronOp(st.num_time, st.num_space, terms, corr)


def su_from_indicator(st, values, tol=0.1, cm=1.0, lengths=None):
    """compute_tau -> lowrank_factorize -> assemble_stabilization terms."""
    tau = stab.compute_tau(st.time)
    lr = stab.lowrank_factorize(stab.indicator_for(st, values), tol)
    return stab.assemble_stabilization(tau, lr, st, cm, lengths), lr, tau


def preconditioner(st, T, cm, sigma, consts, lengths=None):
    """solver.py:193-202: FastDiag.build(..., D, a*c1, spatial_data)."""
    sig = np.atleast_1d(np.asarray(sigma, float))
    react = consts["a"] * consts["c1"]
    if sig.size == 1:
        return FastDiag.build(st, T, cm, float(sig[0]), react, lengths=lengths)
    return FastDiag.build(st, T, cm, 1.0, react, sigma=sig, lengths=lengths)


def config_space(cfg, scale=None):
    """Space-time space of a BASELINE config (optionally a reduced mesh)."""
    c = CONFIGS[cfg]
    ne, ne_t = c["ne"], c["ne_t"]
    if scale is not None:
        ne, ne_t = scale
    return make_space_time(c["d"], c["p"], ne, ne_t), c
