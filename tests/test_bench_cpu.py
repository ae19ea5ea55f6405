"""bench.py launch plumbing on CPU: `--gpus 2` without a launcher re-executes
the script under torch.distributed.run with 2 ranks, which exchange their
packed keys (gloo here, NCCL on the GPU box) and agree on the global order;
rank 0 prints one line with n_gpus == 2."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args):
    env = {k: v for k, v in os.environ.items()
           if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR", "MASTER_PORT")}
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       env=env, capture_output=True, text=True, timeout=300)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_gpus_2_spawns_two_ranks():
    line = _run(["--dry-run", "--gpus", "2", "--steps", "2", "--warmup", "1", "--apps", "3001"])
    assert line["n_gpus"] == 2
    assert line["ranks_seen"] == [0, 1]
    assert line["order_ok"] is True
    assert line["steps"] == 2 and line["warmup"] == 1


def test_gpus_1_stays_in_process():
    line = _run(["--dry-run", "--steps", "1", "--warmup", "0", "--apps", "100"])
    assert line["n_gpus"] == 1 and line["ranks_seen"] == [0] and line["order_ok"]
