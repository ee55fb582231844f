"""bench.py's launcher (CPU, no GPU): ``--gpus N`` without a torchrun
environment starts N rank processes itself (RANK / WORLD_SIZE / MASTER_* set,
127.0.0.1 rendezvous); ``--dry-run`` runs them over gloo and checks that the
row partition covers every row once and each rank holds only its own slice.
Without ``--dry-run`` on a box with fewer GPUs than asked it must fail
instead of timing fewer ranks (BASELINE.json: "... at 1/2/4/8 GPU")."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                              "MASTER_PORT")}
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args, capture_output=True, text=True,
                          timeout=timeout, env=env, cwd=ROOT)


@pytest.mark.parametrize("n,cfg,size", [(2, "3", 10), (3, "4", 4), (4, "2b", 12)])
def test_self_launch_dry_run(n, cfg, size):
    p = _run(["--gpus", str(n), "--dry-run", "--config", cfg, "--size", str(size)])
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1                      # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["covers"] and d["nnz_P_total_ok"]
    assert len(set(d["pids"])) == n             # n distinct processes
    assert all(v > 0 for v in d["nnz_P_per_rank"])


def test_more_gpus_than_visible_fails():
    import torch
    have = torch.cuda.device_count() if torch.cuda.is_available() else 0
    want = max(2, have + 1)
    p = _run(["--gpus", str(want), "--config", "3", "--size", "8", "--steps", "1"])
    assert p.returncode != 0
    d = json.loads([l for l in p.stdout.splitlines() if l.startswith("{")][0])
    assert "error" in d and d["n_gpus"] == want
