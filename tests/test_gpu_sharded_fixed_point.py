"""GPU: the sharded fixed-point driver (sharded.sharded_fixed_point_solve: z-slab potential solve with
halo exchanges, all-to-all P^-1 and all-reduced GMRES; replicated indicator and recovery solve) at 2
and 4 ranks against the single-rank driver, with Spline Upwind and with the u0 lifting.

gpurun gives one GPU, so the ranks share cuda:0 and talk through gloo with host-staged collectives
(MI_DIST_BACKEND=gloo); the orchestration, the exchanged layouts and the per-rank contexts are those
of the NCCL run.
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n, extra):
    env = dict(os.environ, MI_DIST_BACKEND="gloo")
    script = os.path.join(ROOT, "tools", "sharded_solve.py")
    if n == 1:
        cmd = [sys.executable, script, "--single"] + extra
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
               "--master-addr", "127.0.0.1", "--master-port", str(29640 + n), script] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    for ln in r.stdout.splitlines():
        if ln.startswith("{"):
            return json.loads(ln)
    raise AssertionError(r.stdout[-2000:])


@pytest.mark.parametrize("extra", [[], ["--u0"], ["--stab", "off", "--p", "3", "--ne", "4", "4", "10", "--ne-t", "6"]],
                         ids=["su_pulse", "su_u0", "galerkin_p3"])
def test_sharded_fixed_point_matches_single_rank(extra):
    ref = _run(1, extra)
    for n in (2, 4):
        got = _run(n, extra)
        assert got["sweeps"] == ref["sweeps"], n
        assert got["gmres"] == ref["gmres"], n
        assert got["pcg"] == ref["pcg"], n
        for key in ("u", "w"):
            a, b = np.asarray(got[key]), np.asarray(ref[key])
            assert np.linalg.norm(a - b) / np.linalg.norm(b) < 1e-10, (n, key)
        np.testing.assert_allclose(got["increments"], ref["increments"], rtol=1e-8)
