"""bench.py --gpus N launches its own N ranks (torch.distributed.run on 127.0.0.1)
when no launcher set WORLD_SIZE; the --dry-run path runs the whole multi-rank
plumbing on CPU with gloo: rendezvous, per-rank C5 shards with no collective on the
step, barrier + max-over-ranks timing, and ONE JSON line from rank 0."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*argv, timeout=240):
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    env["CUDA_VISIBLE_DEVICES"] = ""
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *argv], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, p.stdout  # exactly one JSON line, from rank 0
    return json.loads(lines[0]), p.stderr


@pytest.mark.parametrize("n", [1, 2])
def test_bench_gpus_n_spawns_n_ranks(n):
    res, err = _run("--gpus", str(n), "--dry-run", "--steps", "3", "--warmup", "3")
    assert res["dry_run"] is True
    assert res["n_gpus"] == n
    assert res["comm"]["nranks"] == n
    assert res["comm"]["backend"] == ("gloo" if n > 1 else None)
    assert res["comm"]["collectives_on_hot_path"] == 0
    assert res["shards_cover_batch"] and res["shard_sums_ok"]
    assert len(res["shards"]) == n and res["config"]["global_batch"] == 2048
    if n > 1:
        assert "spawning 2 ranks" in err
