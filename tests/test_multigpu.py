"""Multi-GPU parity (-m gpu, needs >= 2 GPUs): row-sharded layer over 2 GPUs with NCCL all-to-alls
inside libemb vs the serial oracle (tests/mgpu_worker.py, one process per GPU via torchrun)."""
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _ngpu():
    try:
        import torch
        return torch.cuda.device_count()
    except Exception:
        return 0


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("case,shard,exchange", [("c3", "cyclic", "p2p"), ("hot", "cyclic", "p2p"),
                                                 ("c3", "block", "p2p"), ("c3rw", "cyclic", "p2p"),
                                                 ("c3full", "cyclic", "p2p"), ("c3", "cyclic", "nccl"),
                                                 ("gen", "cyclic", "p2p"), ("hot", "block", "nccl"),
                                                 ("edge", "cyclic", "p2p"), ("edge", "block", "nccl")])
def test_two_gpu_row_sharded_parity(case, shard, exchange):
    """exchange: "p2p" = the peer-memory exchange kernels (default); "nccl" = the v1 grouped
    send/recv exchange (EMB_EXCHANGE=nccl). Case "gen" has a non-monotone slot -> table map, which
    takes the general sort path and the NCCL exchange whatever `exchange` says."""
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs")
    from paper_2112_02752_b200 import build
    build.build()
    env = dict(os.environ, EMB_MGPU_CASE=case, EMB_MGPU_SHARD=shard)
    if exchange == "nccl":
        env["EMB_EXCHANGE"] = "nccl"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
