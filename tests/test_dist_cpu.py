"""CPU, world_size 2 over gloo: the host-side logic of the N>1 path.

* the NCCL unique id that rank 0 creates reaches every rank byte-identical
  (S2Reducer's communicator bootstrap, reducer.broadcast_unique_id);
* the distributed decomposition the GPU path implements — local compress,
  SUM all-reduce of the sketch, OR of the bitmaps (all-gather + OR), replicated
  decode ÷ W — equals the reference's in-process sparse_merge list fold
  (sparse.py:174-196), using the oracle for the arithmetic.
"""
import os
import socket

import numpy as np
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys

    import torch
    import torch.distributed as dist

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from oracle import s2_oracle as o
        from paper_2110_02140_b200.reducer import broadcast_unique_id

        uid = broadcast_unique_id(rank)
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        assert len(uid) == 128 and all(i == uid for i in ids)

        d, rows, cols = 50_000, 3, 997
        g = o.synthetic_gradient(d, 0.02, rank, kind="normal")
        p = o.compress(g, g != 0, rows, cols, 0)
        table = torch.from_numpy(p.table.copy())
        dist.all_reduce(table, op=dist.ReduceOp.SUM)  # K3a
        words = torch.from_numpy(o.mask_words(p.flags).view(np.int32).copy())
        gathered = [torch.empty_like(words) for _ in range(world)]
        dist.all_gather(gathered, words)  # K3b: all-gather ...
        union = np.bitwise_or.reduce(np.stack([w.numpy().view(np.uint32) for w in gathered]), axis=0)  # ... + OR
        merged = o.Payload(d, o.words_to_flags(union, d), table.numpy(), rows, cols, 0, workers=world)
        out = o.decompress(merged)

        ref_ps = [o.compress(gr, gr != 0, rows, cols, 0) for gr in
                  (o.synthetic_gradient(d, 0.02, r, kind="normal") for r in range(world))]
        ref = o.merge(ref_ps)
        assert np.array_equal(merged.flags, ref.flags)
        np.testing.assert_allclose(merged.table, ref.table, rtol=0, atol=1e-12)
        np.testing.assert_allclose(out, o.decompress(ref), rtol=0, atol=1e-12)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_decomposition():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(60)
    assert res == {0: "ok", 1: "ok"}, res
