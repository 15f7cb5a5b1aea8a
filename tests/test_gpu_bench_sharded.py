"""GPU: the N > 1 bench path (bench.py run_sharded: p-plane halo exchange, z-slab operator,
two all-to-all transposes in P^-1) end to end at 2 and 3 ranks.

gpurun gives one GPU, so the ranks share cuda:0 and talk through gloo with host-staged collectives
(MI_DIST_BACKEND=gloo; the kernels never wait on one another).  |P^-1 A x| summed over the ranks'
slabs must equal the single-rank value: the sharded orchestration, the layouts of every exchanged
block and the per-rank CUDA contexts are those of the 8-GPU NCCL run.
"""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["--steps", "1", "--warmup", "1", "--skip-extras", "--no-cpu-baseline", "--ne", "12", "--ne-t", "16"]


def _line(out):
    for ln in out.splitlines():
        if ln.startswith("{"):
            return json.loads(ln)
    raise AssertionError("no JSON line in:\n" + out[-2000:])


def _run(n):
    env = dict(os.environ, MI_DIST_BACKEND="gloo")
    if n == 1:
        cmd = [sys.executable, "bench.py", "--force-sharded"] + ARGS
    else:
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(n),
               "--master-addr", "127.0.0.1", "--master-port", str(29610 + n), "bench.py", "--gpus", str(n)] + ARGS
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    return _line(r.stdout)


def test_sharded_bench_path_matches_single_rank():
    ref = _run(1)
    for n in (2, 3):
        line = _run(n)
        assert line["n_gpus"] == n and line["sharding"]["backend"] == "gloo"
        assert abs(line["z_norm"] - ref["z_norm"]) <= 1e-12 * ref["z_norm"], (n, line["z_norm"], ref["z_norm"])
