"""Multi-GPU parity (a14): distributed lists == single-GPU lists restricted to
each rank's targets (bit-exact), near field bit-identical, full field within
1e-6 of the single-GPU run and 1e-3 of the closed form.  Needs >= 2 GPUs
(skipped otherwise); the host logic is covered on CPU by test_partition_gloo."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    import torch
    return torch.cuda.device_count() if torch.cuda.is_available() else 0


def _launch(world, mode, side, port):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", str(world),
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "tests", "mgpu_check.py"), "--side", str(side), "--mode", mode]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    print(json.dumps(res))
    assert res["ok"], res


@pytest.mark.parametrize("mode", ["tiled", "refined"])
@pytest.mark.parametrize("world", [2, 4, 8])
def test_let_forest_equals_single_gpu(world, mode):
    """a14: local trees + LET-MAC exchange; lists (as cell tuples) bit-exact
    against one GPU restricted to each rank's targets, fallback 0."""
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    _launch(world, mode, 16, 29500 + world)


@pytest.mark.parametrize("mode", ["orb", "orb_cloud"])
@pytest.mark.parametrize("world", [2, 3, 4])
def test_orb_partition(world, mode):
    """NEXT-3: ORB recursive multisection of arbitrary per-rank
    subsets (non-power-of-2 rank counts, clustered cloud), balanced to one
    particle, results in every rank's caller order."""
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    _launch(world, mode, 20, 29520 + world)


@pytest.mark.parametrize("world", [2, 3])
def test_multi_gpu_time_step(world):
    """NEXT-1 on several GPUs: fmm_step with the ORB partition reused
    between the RK2 stages equals the single-GPU step and the oracle's RK2."""
    if _ngpu() < world:
        pytest.skip("needs %d GPUs" % world)
    _launch(world, "step", 16, 29540 + world)


@pytest.mark.parametrize("mode", ["uneven", "leaf_first"])
def test_let_forest_edge_cases(mode):
    """a14 edge cases on 2 GPUs: a rank with no particles and uneven cuts through
    cells (partition 0, jittered lattice), and the leaf-first traversal (Z11)
    whose LET carries the bodies of every visited leaf; fallback 0, full field
    against one GPU and the closed form."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    _launch(2 if mode == "leaf_first" else 3 if _ngpu() >= 3 else 2, mode, 12, 29560 + len(mode))
