"""bench.py's multi-rank harness on CPU: `--gpus 2 --stub --backend gloo`
re-launches itself under torch.distributed.run with two ranks, splits the
global batch B/N (strong scaling), all-reduces the per-step gradient, and
reports the true world size (no GPU: a NumPy stand-in evaluator)."""

import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    env = dict(os.environ, MASTER_ADDR="127.0.0.1", OMP_NUM_THREADS="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), *args], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_spawns_two_ranks_and_splits_the_batch():
    line = _run("--gpus", "2", "--stub", "--backend", "gloo", "--steps", "3", "--warmup", "1")
    assert line["n_gpus"] == 2
    assert line["scaling"] == "strong"
    assert line["config"]["global_batch"] == 4096
    assert line["config"]["batch_per_gpu"] == 2048
    d = line["grad_digest_per_rank"]
    assert len(d) == 2 and d[0] == d[1]          # every rank holds the same all-reduced gradient


def test_bench_single_rank_stub_matches_two_rank_gradient():
    one = _run("--gpus", "1", "--stub", "--backend", "gloo", "--steps", "2", "--warmup", "1")
    two = _run("--gpus", "2", "--stub", "--backend", "gloo", "--steps", "2", "--warmup", "1")
    assert one["n_gpus"] == 1 and one["config"]["batch_per_gpu"] == 4096
    # the stand-in rows are integer-valued, so the cross-rank sum of the two
    # half-batch partial gradients equals the one-rank gradient exactly
    assert two["grad_digest_per_rank"][0] == one["grad_digest_per_rank"][0]
