"""bench.py end to end on the GPU: the one-GPU JSON contract, and the N>1 path
(torchrun, chains sharded per rank, max-over-ranks timing, the end-of-search
exchange) with two ranks sharing the one available GPU over gloo."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _last_json(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert lines, out[-2000:]
    return json.loads(lines[-1])


def test_bench_single_gpu_line_has_the_contract_keys():
    cmd = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--chains", "256", "--budget-ms", "20",
           "--extra", "alexnet", "--no-cpu-baseline", "--py-ref-seconds", "0"]
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, check=True).stdout
    d = _last_json(out)
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks", "full_eval", "evals_by_kind"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["value"] > 0 and d["chain_failures"] == 0
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["e2e"]["d2h_bytes_per_step"] > 0
    assert 0 < d["roofline"]["frac"] < 1
    assert d["configs"]["alexnet"]["value"] > 0 and d["configs"]["alexnet"]["failures"] == 0


def test_bench_two_ranks_share_one_gpu():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--gpus", "2", "--steps", "2",
           "--warmup", "3", "--chains", "128", "--budget-ms", "20", "--extra", "none", "--no-cpu-baseline",
           "--py-ref-seconds", "0"]
    env = {**os.environ, "PS_BENCH_BACKEND": "gloo"}
    out = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=900, check=True, env=env).stdout
    d = _last_json(out)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["chain_failures"] == 0
    assert d["scaling"] == "weak"
    # the winner is a chain of one of the two ranks' blocks (0..255)
    assert 0 <= d["best_chain"] < 256 and d["best_makespan"] > 0
