"""Multi-process (gloo, world_size 2 and 3, CPU) tests of the band-mode host
logic in paper_2212_00488_b200/dist.py: band geometry, the one-step P2P halo
exchange, the global rule-(d) patch.  The per-band compute is the CPU oracle
(test infrastructure) so the test runs anywhere; the assembled bands must equal
the full-frame oracle bit for bit (DESIGN.md §6 correctness criterion)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import dist as sdist
from paper_2212_00488_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _oracle_band(Lb, Rb, D, K, w_y, rank, bands, H):
    """Band compute with the oracle + the same rule-(d) patch dist.py applies."""
    import torch
    import torch.distributed as dist
    p = oracle.params(k_scale=K, w_y=w_y)
    r = oracle.pipeline(Lb, Rb, D, p, "fixed", stages=("median", "fill", "out"))
    b = bands[rank]
    Hs = H // K
    s0 = b.r0 // K
    med = r["median"]
    valid = med != 255
    own = slice(b.ys0 - s0, b.ys1 - s0)
    has = valid[own].any(axis=1).astype(np.int64)
    first = np.array([row[np.argmax(v)] if v.any() else -1 for row, v in zip(med[own], valid[own])])
    last = np.array([row[len(v) - 1 - np.argmax(v[::-1])] if v.any() else -1
                     for row, v in zip(med[own], valid[own])])
    summ = sdist.gather_row_summaries(np.stack([has, first, last]), b, Hs, dist, "cpu")
    rows, vals = sdist.rule_d_patches(summ, b, K, med.shape[0])
    out = r["out"]
    if len(rows):
        fill = r["fill"].copy()
        for y, v in zip(rows, vals):
            fill[y] = v
        out = fill if K == 1 else oracle.scale_up(fill, Lb, K, p.t_fill)
    return out[b.o0 - b.r0:b.o1 - b.r0]


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, D, K, w_y, kind = case
        if kind == "scene":
            L, R, _ = synth.scene(W, H, D, seed=11)
        else:  # unrelated noise: many rows without a single GCP (rule (d))
            L, R = synth.random_pair(W, H, seed=5, levels=256)
        bands = sdist.band_plan(H, world, K, w_y)
        b = bands[rank]
        a0, a1 = sdist.owned_rows(b, H, K)
        Lown = torch.from_numpy(L[a0:a1].copy())
        Rown = torch.from_numpy(R[a0:a1].copy())
        Lb, Rb = sdist.exchange_halos(Lown, Rown, bands, rank, H, K, dist)
        assert np.array_equal(Lb.numpy(), L[b.r0:b.r1]) and np.array_equal(Rb.numpy(), R[b.r0:b.r1])
        mine = _oracle_band(Lb.numpy(), Rb.numpy(), D, K, w_y, rank, bands, H)
        parts = [None] * world
        dist.all_gather_object(parts, (b.o0, b.o1, mine))
        if rank == 0:
            full = oracle.pipeline(L, R, D, oracle.params(k_scale=K, w_y=w_y), "fixed",
                                   stages=("out",))["out"]
            got = np.zeros_like(full)
            for o0, o1, part in parts:
                got[o0:o1] = part
            q.put(bool(np.array_equal(got.view(np.uint32), full.view(np.uint32))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (160, 120, 32, 2, 31, "scene")),
    (3, (96, 150, 24, 1, 7, "scene")),
    (2, (24, 60, 16, 1, 3, "noise")),
    (3, (20, 62, 20, 2, 4, "noise")),
    (3, (10, 90, 16, 2, 1, "noise")),  # rows 26..30 have no GCP: only the global patch is right
])
def test_bands_equal_full_frame(world, case):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10)


def test_band_plan_covers_and_aligns():
    for H, P, K in ((992, 8, 2), (991, 3, 2), (375, 4, 1), (1984, 8, 2)):
        bands = sdist.band_plan(H, P, K)
        assert bands[0].o0 == 0 and bands[-1].o1 == H
        for a, b in zip(bands, bands[1:]):
            assert a.o1 == b.o0 and a.ys1 == b.ys0
        for b in bands:
            assert b.r0 % K == 0 and b.r0 <= b.o0 and b.r1 >= b.o1
    with pytest.raises(ValueError):
        sdist.band_plan(10, 8, 2)


def test_rule_d_patch_values():
    # rows 0..5: valid at 1 (values 3/7) and 4 (values 9/2)
    has = np.array([0, 1, 0, 0, 1, 0])
    first = np.array([-1, 3, -1, -1, 9, -1])
    last = np.array([-1, 7, -1, -1, 2, -1])
    b = sdist.Band(0, 0, 6, 0, 6, 0, 6)
    rows, vals = sdist.rule_d_patches(np.stack([has, first, last]), b, 1, 6)
    assert rows.tolist() == [0, 2, 3, 5] and vals.tolist() == [3.0, 7.0, 7.0, 2.0]
    none = sdist.rule_d_patches(np.zeros((3, 4), int), sdist.Band(0, 0, 4, 0, 4, 0, 4), 1, 4)
    assert none[1].tolist() == [0.0] * 4


def test_stream_slices_partition():
    for n, P in ((256, 8), (10, 3), (7, 7)):
        got = sorted(i for r in range(P) for i in sdist.stream_slice(n, P, r))
        assert got == list(range(n))
