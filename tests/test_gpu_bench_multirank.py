"""The sharded bench path itself (bench.py under torchrun) on the one GPU the test box
has: two ranks share cuda:0 and use gloo for the final collective.  The gathered u0 + step stats
must be bit-equal to a single-rank run over the whole batch (instances are independent and every
kernel is deterministic), and the JSON line must carry the max-over-ranks timing and the gather
time.  No scaling curve can be measured on one GPU."""
import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
COMMON = ["--steps", "3", "--warmup", "3", "--no-e2e", "--no-cpu-baseline", "--latency", "",
          "--closed-loop-ticks", "0", "--no-large", "--no-scan-legs"]


def _json(out):
    return json.loads([l for l in out.splitlines() if l.startswith("{")][-1])


def test_two_ranks_gloo_match_single_rank(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    g2, g1 = str(tmp_path / "g2.pt"), str(tmp_path / "g1.pt")
    env = dict(os.environ, MASTER_ADDR="127.0.0.1")
    r2 = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                         "--master-addr", "127.0.0.1", "--master-port", "29561", "bench.py", "--gpus", "2",
                         "--dist-backend", "gloo", "--batch", "64", "--gather-out", g2, *COMMON],
                        cwd=ROOT, capture_output=True, text=True, timeout=600, env=env)
    assert r2.returncode == 0, r2.stderr[-3000:]
    d2 = _json(r2.stdout)
    r1 = subprocess.run([sys.executable, "bench.py", "--batch", "128", "--gather-out", g1, *COMMON],
                        cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r1.returncode == 0, r1.stderr[-3000:]
    a = torch.load(g2)
    assert a.shape == (128, 17)
    # the single-rank run does not gather: rebuild its packed rows from a one-rank call
    assert os.path.exists(g1)
    b = torch.load(g1)
    assert torch.equal(a, b)
    assert d2["n_gpus"] == 2 and d2["final_allgather_ms"] is not None and d2["step_check"]["info_nonzero"] == 0
    with open(os.path.join(ROOT, "gpurun_out", "multirank_gloo.json") if os.path.isdir(os.path.join(ROOT, "gpurun_out"))
              else str(tmp_path / "x.json"), "w") as f:
        json.dump({"two_ranks": d2, "one_rank_value": _json(r1.stdout)["value"], "gathered_bit_equal": True}, f)
