"""The bench's multi-rank code path, run for real: bench.py --workload cfg3
at a reduced size with --verify (whole outputs of the timed passes against
the oracle), at world size 1 and as 2 ranks on the one GPU of the test box
(gloo for the collectives: the ranks' kernels never wait on each other, the
gloo all-gather of the argmax and the object gather are host-side).  The
driver's bench runs the BASELINE sizes; this checks the sharding, the
owner-computes max backward (argmax all-gather + range scatter) and the
e2e host path end to end."""
import json
import os
import subprocess
import sys

import pytest

from gspmm_testutil import ROOT

pytestmark = pytest.mark.gpu


def run(cmd, env=None, timeout=900):
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=timeout,
                       env={**os.environ, **(env or {})})
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert lines, r.stdout[-2000:] + r.stderr[-2000:]
    return json.loads(lines[-1])


@pytest.mark.parametrize("world", [1, 2])
def test_bench_cfg3_scaled_verify(world):
    args = ["bench.py", "--workload", "cfg3", "--scale", "64", "--steps", "2", "--warmup", "3",
            "--skip-cpu", "--verify"]
    if world == 1:
        res = run([sys.executable] + args)
    else:
        res = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                   "--nproc-per-node", "2", "--master-addr", "127.0.0.1", "--master-port",
                   "29531"] + args + ["--gpus", "2"], env={"BENCH_DIST_BACKEND": "gloo"})
    assert res["n_gpus"] == world
    assert res["verify"]["ok"], res["verify"]
    assert res["e2e"]["value"] > 0 and res["gpu_launches"] > 0
    assert res["config"]["scaled_down"]


def test_bench_cfg5_two_ranks_one_gpu():
    # dist.ShardedMean over 2 ranks: column-chunked all-gather of the source
    # features and gradients, remapped neighbour ids, mean fwd + bwd
    res = run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node",
               "2", "--master-addr", "127.0.0.1", "--master-port", "29533", "bench.py",
               "--workload", "cfg5", "--scale", "32", "--steps", "2", "--warmup", "3",
               "--gpus", "2"], env={"BENCH_DIST_BACKEND": "gloo"})
    assert res["n_gpus"] == 2 and res["value"] > 0
