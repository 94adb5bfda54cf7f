"""CPU test of bench.py's multi-GPU launcher (world_size 2, gloo).

`python bench.py --gpus N` started without torchrun must start N ranks
itself (re-exec under torch.distributed.run, rendezvous on 127.0.0.1) with
correct RANK / LOCAL_RANK / WORLD_SIZE, and the exchange step -- the exact
integer moment merge paper_1010_2438_b200.dist.allreduce_stats -- must sum
the ranks' moments exactly (sumsq carries across the 64-bit word).  The
hidden --selftest-dist mode runs that path on CPU (gloo) with synthetic
per-rank moments; no GPU and no oracle involved."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(n):
    env = {k: v for k, v in os.environ.items() if k not in ("RANK", "WORLD_SIZE", "LOCAL_RANK", "MASTER_ADDR",
                                                             "MASTER_PORT")}
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--selftest-dist"],
                       capture_output=True, text=True, timeout=300, env=env, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [json.loads(x) for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    return lines[0]


def test_launcher_starts_two_ranks_and_merges_exactly():
    d = _run(2)
    assert d == {"selftest": "dist", "world_size": 2, "ranks_env_ok": True, "merge_exact": True,
                 "comm_nranks_ok": True}


def test_launcher_three_ranks():
    d = _run(3)
    assert d["world_size"] == 3 and d["ranks_env_ok"] and d["merge_exact"] and d["comm_nranks_ok"]
