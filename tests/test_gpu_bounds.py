"""Out-of-bounds write checks by guard bands (compute-sanitizer is closed on this GPU pool).

Every device output of the C ABI is placed inside a larger allocation whose head and tail
(4 KB each) hold a sentinel pattern; after the call the guards must be untouched and the
interior must still match the oracle.  Shapes are the ragged ones that exercise tail paths:
dims not a multiple of 4 / 32 / 1024, one-element vectors, block sizes that leave empty or
short tail blocks, non-power-of-two widths, rows 1..16, and W-rank exchanges whose arenas
are guarded the same way.
"""
import ctypes

import numpy as np
import pytest

from oracle import s2_oracle as o

pytestmark = pytest.mark.gpu
GUARD = 4096  # bytes on each side
SENT = 0x5A5A5A5A


class Guarded:
    """A device buffer of `nbytes` with sentinel guard bands; .ptr is 256-byte aligned."""

    def __init__(self, nbytes, fill=0):
        import torch

        self.nbytes = int(nbytes)
        n = (2 * GUARD + self.nbytes + 3) // 4
        self.buf = torch.full((n,), SENT, dtype=torch.int32, device="cuda")
        self.inner = self.buf[GUARD // 4: GUARD // 4 + (self.nbytes + 3) // 4]
        self.inner.fill_(fill)
        self.ptr = ctypes.c_void_p(self.inner.data_ptr())

    def view(self, dtype, count):
        return self.inner.view(dtype)[:count]

    def intact(self) -> bool:
        g = GUARD // 4
        head, tail = self.buf[:g], self.buf[g + (self.nbytes + 3) // 4:]
        return bool((head == SENT).all()) and bool((tail == SENT).all())


SHAPES = [(1, 1, 3, 2), (33, 33, 3, 7), (1025, 1025, 5, 97), (100_003, 100_003, 3, 1667),
          (100_003, 3_126, 3, 1667), (4_099, 4_098, 16, 31), (65_537, 7, 2, 4096), (1_000_000, 1_000_000, 1, 16384)]


@pytest.mark.parametrize("dim,nb,rows,cols", SHAPES)
def test_single_gpu_ops_stay_in_bounds(dim, nb, rows, cols):
    import torch

    from paper_2110_02140_b200._lib import S2_MASK_GIVEN, S2_MASK_NONZERO, check, lib
    from paper_2110_02140_b200.sketch import Plan

    rng = np.random.default_rng(dim + nb)
    g = ((rng.random(dim) < 0.05) * rng.integers(-50, 51, dim)).astype(np.float32)
    if dim == 1:
        g[0] = 3.0
    plan = Plan(dim, nb, rows, cols, 7)
    st = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    words = plan.words
    gb = Guarded(4 * dim)
    gb.view(torch.float32, dim).copy_(torch.from_numpy(g))
    bm = Guarded(4 * words)
    tab = Guarded(4 * rows * cols)
    cnt = Guarded(8 * 4)
    out = Guarded(4 * dim)
    check(lib.s2_compress(plan.handle, gb.ptr, bm.ptr, tab.ptr, S2_MASK_NONZERO, cnt.ptr, st))
    check(lib.s2_decode(plan.handle, bm.ptr, tab.ptr, 3, out.ptr, st))
    flags = o.nonzero_flags(g, nb)
    ref = o.compress(g, flags, rows, cols, 7)
    ref.workers = 3
    torch.cuda.synchronize()
    assert np.array_equal(bm.view(torch.int32, words).cpu().numpy().view(np.uint32), o.mask_words(flags))
    assert np.array_equal(tab.view(torch.float32, rows * cols).cpu().numpy(), ref.table.reshape(-1).astype(np.float32))
    assert np.array_equal(out.view(torch.float32, dim).cpu().numpy(), o.decompress(ref).astype(np.float32))
    # given mask (MODE 2), compaction, sketch insert/query, union, table sum, block top-k
    gflags = rng.random(nb) < 0.5
    gm = Guarded(4 * words)
    gm.view(torch.int32, words).copy_(torch.from_numpy(o.mask_words(gflags).view(np.int32)))
    tab2 = Guarded(4 * rows * cols)
    check(lib.s2_compress(plan.handle, gb.ptr, gm.ptr, tab2.ptr, S2_MASK_GIVEN, cnt.ptr, st))
    nsel = int(o.selected_indices(gflags, dim).size)
    scratch = Guarded(int(lib.s2_compact_scratch_bytes(plan.handle)))
    count = Guarded(8)
    idx = Guarded(8 * max(nsel, 1))
    val = Guarded(4 * max(nsel, 1))
    check(lib.s2_compact(plan.handle, gm.ptr, None, idx.ptr, None, count.ptr, scratch.ptr, st))
    nz = int((g[o.selected_indices(gflags, dim)] != 0).sum())
    idx2 = Guarded(8 * max(nz, 1))
    check(lib.s2_compact(plan.handle, gm.ptr, gb.ptr, idx2.ptr, val.ptr, count.ptr, scratch.ptr, st))
    qout = Guarded(4 * max(nz, 1))
    tab3 = Guarded(4 * rows * cols)
    check(lib.s2_sketch_insert(plan.handle, idx2.ptr, val.ptr, nz, tab3.ptr, st))
    check(lib.s2_sketch_query(plan.handle, idx2.ptr, nz, tab3.ptr, qout.ptr, st))
    stacked = Guarded(4 * words * 3)
    un = Guarded(4 * words)
    check(lib.s2_bitmap_or(words, stacked.ptr, 3, un.ptr, st))
    tstack = Guarded(4 * rows * cols * 2)
    tsum = Guarded(4 * rows * cols)
    check(lib.s2_table_sum(rows * cols, tstack.ptr, 2, tsum.ptr, st))
    k = max(1, nb // 3)
    tks = Guarded(int(lib.s2_block_topk_scratch_bytes(plan.handle)))
    tkm = Guarded(4 * words)
    check(lib.s2_block_topk(plan.handle, gb.ptr, k, tkm.ptr, tks.ptr, st))
    torch.cuda.synchronize()
    assert np.array_equal(tab2.view(torch.float32, rows * cols).cpu().numpy(),
                          o.compress(g, gflags, rows, cols, 7).table.reshape(-1).astype(np.float32))
    assert np.array_equal(idx.view(torch.int64, nsel).cpu().numpy(), o.selected_indices(gflags, dim))
    assert np.array_equal(tkm.view(torch.int32, words).cpu().numpy().view(np.uint32),
                          o.mask_words(o.block_topk(g, nb, k)))
    for b in (gb, bm, tab, cnt, out, gm, tab2, scratch, count, idx, val, idx2, qout, tab3, stacked, un, tstack, tsum,
              tks, tkm):
        assert b.intact(), "write outside an output buffer"


@pytest.mark.parametrize("W", [2, 5, 8])
def test_reduce_and_exchange_stay_in_bounds(W):
    """s2_reduce at W = 1 with a guarded output, and the W-rank exchange with guarded arenas."""
    import torch

    from paper_2110_02140_b200._lib import S2_COMM_EXTERNAL, check, lib, ptr
    from paper_2110_02140_b200.sketch import Plan

    dim, rows, cols = 300_007, 3, 4099
    grads = [o.synthetic_gradient(dim, 0.02, r, kind="int") for r in range(W)]
    plans = [Plan(dim, dim, rows, cols, 0) for _ in range(W)]
    for r, p in enumerate(plans):
        check(lib.s2_comm_set_options(p.handle, 4, 20.0))
        check(lib.s2_comm_init_mode(p.handle, W, r, None, S2_COMM_EXTERNAL))
    nbytes = int(lib.s2_p2p_arena_bytes(plans[0].handle, W))
    arenas = [Guarded(nbytes) for _ in range(W)]
    bases = (ctypes.c_uint64 * W)(*[a.ptr.value for a in arenas])
    for p in plans:
        check(lib.s2_comm_attach(p.handle, bases, W))
    outs = [Guarded(4 * dim) for _ in range(W)]
    gt = [torch.from_numpy(x).cuda() for x in grads]
    streams = [torch.cuda.Stream() for _ in range(W)]
    torch.cuda.synchronize()
    for _ in range(3):
        for p, x, o_, s in zip(plans, gt, outs, streams):
            check(lib.s2_reduce(p.handle, ptr(x), o_.ptr, None, ctypes.c_void_p(s.cuda_stream)))
    torch.cuda.synchronize()
    want = o.decompress(o.merge([o.compress(x, x != 0, rows, cols, 0) for x in grads])).astype(np.float32)
    for o_ in outs:
        assert np.array_equal(o_.view(torch.float32, dim).cpu().numpy(), want)
    for b in arenas + outs:
        assert b.intact(), "write outside an arena or output"
