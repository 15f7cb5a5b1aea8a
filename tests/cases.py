"""Shared helpers: load golden fixtures and rebuild the oracle objects for them."""

import os

import numpy as np

from oracle import problem, stab
from oracle.splines import make_space_time

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
CASES = ["case_2d_p2", "case_3d_p3", "case_2d_aniso", "case_1d_p1", "case_cfg1", "case_3d_p2_front"]
RM = {"c1": 0.26, "a": 0.13, "c2": 0.1}


def load(name):
    z = np.load(os.path.join(GOLDEN, name + ".npz"))
    return {k: z[k] for k in z.files}


def space_of(g):
    return make_space_time(int(g["d"]), int(g["p"]), [int(v) for v in g["ne"]], int(g["ne_t"]))


def sigma_of(g):
    s = np.atleast_1d(g["sigma"])
    return float(s[0]) if s.size == 1 else s


def oracle_objects(g):
    """(st, op_a, op_b, P, su_terms) rebuilt with the oracle for fixture g."""
    st = space_of(g)
    T = float(g["T"])
    su, lr, _ = problem.su_from_indicator(st, g["theta"], float(g["su_tol"]))
    op_a = problem.operator_terms(st, T, 1.0, sigma_of(g), RM, su_terms=su)
    op_b = problem.operator_terms(st, T, 1.0, sigma_of(g), RM, g["u"], g["w"], su_terms=su)
    P = problem.preconditioner(st, T, 1.0, sigma_of(g), RM)
    return st, op_a, op_b, P, su, lr
