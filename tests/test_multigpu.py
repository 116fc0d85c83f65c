"""Multi-GPU parity (-m gpu, needs >= 2 GPUs): the row-sharded layer with one process per GPU (libemb's
peer-memory exchange between processes over CUDA IPC mappings) vs the serial oracle
(tests/mgpu_worker.py via torchrun). The same exchange with all ranks in one process (any number of
GPUs, including one) is tests/test_group_parity.py."""
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


@pytest.mark.parametrize("case,shard,prefetch", [
    ("c3", "cyclic", 0), ("hot", "cyclic", 0), ("c3", "block", 0), ("c3rw", "cyclic", 0), ("c3full", "cyclic", 0),
    ("gen", "cyclic", 0), ("hot", "block", 0), ("edge", "cyclic", 0), ("edge", "block", 0),
    # the next step's sort + route prefetched during each backward (emb_lookup_prefetch at W > 1)
    ("c3", "cyclic", 1), ("c3full", "cyclic", 1), ("edge", "block", 1)])
def test_two_gpu_row_sharded_parity(case, shard, prefetch):
    if _ngpu() < 2:
        pytest.skip("needs 2 GPUs (the one-GPU equivalent is tests/test_group_parity.py)")
    from paper_2112_02752_b200 import build
    build.build()
    env = dict(os.environ, EMB_MGPU_CASE=case, EMB_MGPU_SHARD=shard, EMB_MGPU_PREFETCH=str(prefetch))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), os.path.join(ROOT, "tests", "mgpu_worker.py")]
    for _ in range(3):  # a fresh port per attempt: the rendezvous port can be taken between probe and bind
        cmd[cmd.index("--master-port") + 1] = str(_port())
        r = subprocess.run(cmd, env=env, capture_output=True, text=True, timeout=900)
        if "EADDRINUSE" not in r.stderr:
            break
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-4000:]
