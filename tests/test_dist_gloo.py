"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the partition
and halo planners of libqswg drive an emulated row-sharded SpMV whose result
must equal the single-process product exactly where halos were received."""
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytest.importorskip("paper_2003_02450_b200.api")


@pytest.mark.parametrize("world", [2, 3])
def test_row_sharded_spmv_with_planned_halos(world):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--standalone", "--local-addr", "127.0.0.1",
           "--nproc-per-node", str(world), os.path.join(ROOT, "tests", "dist_worker.py")]
    env = dict(os.environ, OMP_NUM_THREADS="1", MASTER_ADDR="127.0.0.1")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count("ok=True") == 4, r.stdout
