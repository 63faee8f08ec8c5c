"""bench.py's multi-GPU entry point (driver contract: ``bench.py --gpus N``) on
CPU: without a torchrun environment it must start N ranks itself; --dry-run
takes the same launch path with gloo and no GPU."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                            "MASTER_PORT")}
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                         timeout=300, env=env, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout  # rank 0 alone prints
    return json.loads(lines[0])


@pytest.mark.parametrize("n", [1, 2])
def test_gpus_flag_starts_n_ranks(n):
    d = _run("--gpus", str(n), "--dry-run")
    assert d["dry_run"] and d["n_gpus"] == n and d["requested"] == n
    assert len({s["pid"] for s in d["shards"]}) == n          # n distinct processes
    assert [s["rank"] for s in d["shards"]] == list(range(n))
    assert d["tiles_range"] and d["workload"] == "cfg5"       # default workload: the 1.35e10 sweep
    assert d["configs"] == 28 ** 7
