"""Multi-GPU reduce (NCCL over NVLink) against the oracle; needs >= 2 GPUs (gpurun --gpus 2)."""
import json
import os
import subprocess
import sys

import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu


def ngpus():
    import torch

    return torch.cuda.device_count()


VARIANTS = {
    "ipc": {},                                 # default: CUDA-IPC arena, pull one-shot (W=2) / push two-shot (W>2)
    "ipc_twoshot": {"S2_P2P_ONESHOT_MAXW": "1"},   # push two-shot at W = 2 too
    "ipc_oneshot": {"S2_P2P_ONESHOT_MAXW": "4"},   # pull one-shot at W = 4
    "pull": {"S2_P2P_PUSH": "0", "S2_P2P_ONESHOT_MAXW": "1"},  # pull two-shot (peers read after the flag)
    "push_oneshot": {"S2_P2P_PUSH": "1"},      # push one-shot
    "nccl": {"S2_AGG": "nccl"},                # NCCL all-reduce + all-gather + OR kernel (north-star literal)
    "graph": {"S2_CHECK_GRAPH": "1"},          # CUDA-graph replay of the whole reduce
    "many": {"S2_CHECK_MANY": "1"},            # pipelined batch (reduce_many, two streams)
    "many_pull": {"S2_CHECK_MANY": "1", "S2_P2P_PUSH": "0", "S2_P2P_ONESHOT_MAXW": "4"},  # ... peers pull
    "many_one_stream": {"S2_CHECK_MANY": "1", "S2_PIPE_STREAMS": "1"},
    "blocks": {"S2_CHECK_NUM_BLOCKS": "62500"},  # block bitmap (b < d, 32 elements per block)
}


@pytest.mark.parametrize("variant", sorted(VARIANTS))
@pytest.mark.parametrize("world", [2, 4, 8])
def test_dist_reduce_parity(world, variant):
    if ngpus() < world:
        pytest.skip(f"needs {world} GPUs")
    port = 29500 + world * 10 + sorted(VARIANTS).index(variant)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.join(ROOT, "tools", "dist_check.py")]
    env = dict(os.environ, **VARIANTS[variant])
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT, env=env)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    line = [x for x in p.stdout.splitlines() if x.startswith("{")][-1]
    rep = json.loads(line)
    assert rep["all_ranks_ok"], rep


def test_ddp_comm_hook_trains():
    """S2 as a DDP comm hook on an embedding model: one bucket without error feedback, and several
    rebuilt buckets with error feedback (casq.ef_step semantics against the merged estimate)."""
    if ngpus() < 2:
        pytest.skip("needs 2 GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr", "127.0.0.1", "--master-port=29590", os.path.join(ROOT, "tools", "ddp_check.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert p.returncode == 0, p.stdout[-3000:] + p.stderr[-3000:]
    rep = json.loads([x for x in p.stdout.splitlines() if x.startswith("{")][-1])
    assert rep["ok"], rep
