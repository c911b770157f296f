"""Uninitialised reads and out-of-bounds writes, without compute-sanitizer
(closed on this GPU pool): tests/poison_worker.py runs every kernel of the path
on small cases twice in fresh processes -- once normally and once with
FMM_POISON=1, where every device buffer the library allocates starts as 0xFF
bytes (NaN / -1) and carries a 4 KB guard zone that is checked after every API
call (common.cuh, devmem.cu).  The two runs must agree bit for bit (the path is
deterministic, test_gpu_edge.py), so any read of memory that no kernel wrote,
and any write just past a buffer's end, fails here.
"""
import os
import subprocess
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(tmp_path, poison):
    out = tmp_path / ("poison.npz" if poison else "plain.npz")
    env = dict(os.environ)
    env["FMM_POISON"] = "1" if poison else "0"
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "poison_worker.py"), str(out)],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    return dict(np.load(out))


@pytest.mark.gpu
def test_poisoned_allocations_and_guard_zones(tmp_path):
    plain = _run(tmp_path, False)
    poison = _run(tmp_path, True)
    assert sorted(plain) == sorted(poison)
    bad = [k for k in plain if not np.array_equal(plain[k], poison[k])]
    assert not bad, bad
    for k, v in plain.items():
        if v.dtype.kind == "f":
            assert np.all(np.isfinite(v)), k
