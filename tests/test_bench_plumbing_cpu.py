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


def test_parity_report_metrics():
    """bench.py's parity object: rel-L2 over the sample, the worst subcarrier (axis 0 for the uplink
    [N][J][U] outputs, axis 1 for the downlink [C][N][J][S]) and hard-bit mismatch counts."""
    import importlib.util
    import numpy as np
    spec = importlib.util.spec_from_file_location("bench_mod", os.path.join(ROOT, "bench.py"))
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    rng = np.random.default_rng(0)
    n = 6
    s = rng.standard_normal((n, 1, 4)) + 1j * rng.standard_normal((n, 1, 4))
    x = rng.standard_normal((n, 1, 4)) + 1j * rng.standard_normal((n, 1, 4))
    b = rng.standard_normal((3, n, 1, 8)) + 1j * rng.standard_normal((3, n, 1, 8))
    h = rng.integers(0, 16, (n, 1, 4)).astype(np.uint8)
    bench._ORACLE_OUT[n] = ((s, h), (x, h), b)
    s_g = s.copy()
    s_g[2] *= 1.01                                        # one subcarrier off by 1%
    h_g = h.copy()
    h_g[0, 0, 0] ^= 1                                     # one hard decision flipped
    b_g = b.copy()
    b_g[:, 4] *= 1.001                                    # subcarrier 4 of every cluster, downlink axis 1
    out = bench.parity_report((s_g, h_g, x, h, b_g), n_sub=n)
    assert abs(out["admm_ul"]["max_subcarrier"] - 0.01) < 1e-12
    assert 0 < out["admm_ul"]["rel_l2"] < 0.01
    assert out["admm_ul"]["hard_mismatch"] == 1 and out["cg_ul"]["hard_mismatch"] == 0
    assert out["cg_ul"]["rel_l2"] == 0.0
    assert abs(out["admm_dl"]["max_subcarrier"] - 0.001) < 1e-12


def test_reference_arm_line():
    """`bench.py --impl reference` (the fp64 oracle on the host, no GPU needed): one JSON line with the
    base contract's keys, the oracle described as the cpu_baseline of this run, and an e2e without copies."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "0", "--ref-subcarriers", "2"], capture_output=True, text=True, timeout=600,
                       cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[-1])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "Gbit/s" and d["higher_is_better"]
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["C"] == 32 and d["config"]["N"] == 1200
