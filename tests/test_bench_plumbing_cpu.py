"""bench.py's multi-rank launcher and rank plumbing on CPU (gloo, world 2): `--gpus 2` outside
torchrun re-executes itself under torch.distributed.run, every rank checks WORLD_SIZE against
--gpus, the unique id is broadcast, clusters are partitioned contiguously and rank
0 prints the max over ranks -- the same code path the GPU run takes, minus the CUDA work."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_bench_relaunches_two_ranks_and_reduces_over_them():
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    env.pop("RANK", None)
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-check"],
                       capture_output=True, text=True, timeout=240, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout                      # rank 0 alone prints
    d = json.loads(lines[0])
    assert d["plumbing"] and d["n_gpus"] == 2
    assert d["max_ms"] == 2.0                             # max over ranks of (1 + rank)
    assert [x["clusters"] for x in d["ranks"]] == [[0, 16], [16, 32]]
    assert all(x["uid_bytes"] == 128 for x in d["ranks"])  # the broadcast id reached every rank


def test_bench_refuses_world_mismatch():
    env = dict(os.environ, RANK="0", WORLD_SIZE="1", LOCAL_RANK="0", MASTER_ADDR="127.0.0.1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--plumbing-check"],
                       capture_output=True, text=True, timeout=120, env=env, cwd=ROOT)
    assert r.returncode != 0 and "WORLD_SIZE=1" in (r.stderr + r.stdout)
