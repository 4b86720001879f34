"""bench.py's N>1 code paths (torchrun, barriers, max-over-ranks timing, one JSON
line from rank 0) with 2 ranks sharing the one GPU of the test box through the
gloo test mode (BENCH_DIST_BACKEND=gloo); the driver's scaling runs use NCCL
with one GPU per rank."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("args", [["--config", "c3"], ["--config", "c5", "--size", "8192"],
                                  ["--config", "c2", "--depth", "20", "--alt-steps", "0",
                                   "--c5-size", "8192"]])
def test_two_rank_bench_prints_one_line(args):
    env = dict(os.environ, BENCH_DIST_BACKEND="gloo", OMP_NUM_THREADS="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(29600 + len(args) * 7 + len(args[1])),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--steps", "2", "--warmup", "3",
           "--no-primitives", "--no-cpu-baseline", *args]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=280, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    assert lines[0]["n_gpus"] == 2 and lines[0]["value"] > 0
