"""bench.py's N > 1 path as real processes (-m gpu).

Two ranks launched by torch.distributed.run, exactly as the driver launches
the scaling run, each running the product's sharded apply with the output
all-gather fused into the GEMM4 (Ozaki CRT) epilogue over CUDA IPC peer
memory. With one visible GPU both ranks share cuda:0 (TCI_BENCH_SAME_DEVICE
= 1, gloo process group: the test harness switches; NCCL refuses two ranks
on one device) -- the IPC export / mapping, the cross-process flag barriers
and the remote stores still run for real. With >= 2 GPUs the same command
runs one rank per GPU over NCCL. Rank 0's gathered output is checked by
bench.py against the oracle on the first and last row of every rank's slab."""
import json
import os
import socket
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(nproc, env_extra, config="cfg2", gather="p2p"):
    env = dict(os.environ, **env_extra)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={nproc}",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", str(nproc),
           "--steps", "2", "--warmup", "1", "--config", config, "--gather", gather, "--alt", "none",
           "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    return json.loads(lines[-1])


def test_bench_two_processes_same_gpu_fused_gather():
    line = _run(2, {"TCI_BENCH_BACKEND": "gloo", "TCI_BENCH_SAME_DEVICE": "1"})
    assert line["n_gpus"] == 2 and line["config"]["gather"] == "p2p", line.get("config")
    assert line["parity"]["rel_frob"] <= 1e-12, line["parity"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("gather", ["p2p", "nccl"])
def test_bench_two_gpus(gather):
    line = _run(2, {}, gather=gather)
    assert line["n_gpus"] == 2
    assert line["parity"]["rel_frob"] <= 1e-12, line["parity"]
