"""bench.py launches its own ranks: `python bench.py --gpus 2` re-executes itself under
torch.distributed.run (one process per GPU).  On a one-GPU box the gloo test backend lets
both ranks share cuda:0 (STAR_BENCH_BACKEND=gloo), which exercises the multi-rank bench
logic — sharded blocks, max-over-ranks timing, per-rank K1 roofline, peer-exchange decode —
end to end.  The numbers of such a run are not a measurement (two ranks time-slice one GPU).
"""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_two_ranks_self_launch():
    env = dict(os.environ, STAR_BENCH_BACKEND="gloo")
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "2", "--warmup", "3",
                        "--no-e2e", "--no-sweep", "--no-cpu-baseline"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0
    assert line["process_group"]["world"] == 2
    assert [p["rank"] for p in line["roofline"]["per_rank"]] == [0, 1]
    assert line["roofline"]["rank"] in (0, 1)
    assert "us_per_token" in line["decode"]["layers32"], line["decode"]["layers32"]


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, WORLD_SIZE="3", RANK="0")
    r = subprocess.run([sys.executable, "bench.py", "--gpus", "2"], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=300)
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr
