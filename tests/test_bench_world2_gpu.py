"""bench.py's world > 1 path end to end on one GPU: `--gpus 2 --host-comm` relaunches itself under
torch.distributed.run with two ranks sharing the GPU, the consensus exchange going through the
library's host allreduce hook over gloo (NCCL refuses two ranks on one device).  Everything else
is what an 8-GPU run executes: the rank plumbing, the timed regions and max-over-ranks
reductions, the per-rank exposed-communication rows, the device-consensus leg (here on the
split path: no peer mapping without NCCL), the world-1 cross-check and the subcarrier-sharded
control -- so a Python fault in those legs cannot first show up on the multi-GPU box."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_world2_host_comm():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    for k in ("RANK", "WORLD_SIZE", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--host-comm", "--steps", "3",
                        "--warmup", "3", "--e2e-steps", "1"], capture_output=True, text=True, timeout=900, env=env,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["schedule"] == "sequential on one stream"
    m = d["multi_gpu"]
    assert m["nccl_comm"] == {"nranks": 2, "rank": 0}
    assert len(m["per_rank"]) == 2 and all(p["allreduce_calls_per_step"] == 15 for p in m["per_rank"])
    assert m["vs_world1"]["ok"], m["vs_world1"]
    assert "ms_per_step" in m["modes"]["control_subcarrier_sharded"]
    dc = m["modes"]["device_consensus"]
    assert "error" in dc or max(dc["rel_l2_vs_nccl"].values()) < 1e-5
    assert d["consensus_rounds_per_step"] == 15 and d["e2e"]["value"] > 0
