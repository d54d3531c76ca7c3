"""Multi-process (gloo, world_size 2 and 3, CPU) tests of the band-mode
plumbing in paper_2212_00488_b200/dist.py: the library's band partition and
halo rules (host functions of the C ABI, no GPU needed), the one-step P2P halo
exchange into the preallocated sub-images, and the MAX all-reduce that
assembles the frame-wide fill summaries.

The per-band compute here is the CPU oracle (test infrastructure), run on the
exchanged sub-image: its own rows must equal the full-frame oracle bit for bit
(the halo covers the dependency cone) except where fill rule (d) needs other
bands' rows, which the test resolves from the all-reduced summaries exactly as
stereo_band_finish does on the GPU (DESIGN.md §6 correctness criterion)."""
import os
import socket

import numpy as np
import pytest

import oracle
from paper_2212_00488_b200 import abi
from paper_2212_00488_b200 import dist as sdist
from paper_2212_00488_b200 import synth


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _summaries(med):
    """(last valid value, first valid value) per row, -1 = none."""
    valid = med != 255
    last = np.array([row[len(v) - 1 - np.argmax(v[::-1])] if v.any() else -1 for row, v in zip(med, valid)])
    first = np.array([row[np.argmax(v)] if v.any() else -1 for row, v in zip(med, valid)])
    return np.stack([last, first], axis=1).astype(np.int32)


def _rule_d_value(summ, y):
    for yy in range(y - 1, -1, -1):
        if summ[yy, 0] >= 0:
            return float(summ[yy, 0])
    for yy in range(y + 1, summ.shape[0]):
        if summ[yy, 1] >= 0:
            return float(summ[yy, 1])
    return 0.0


def _worker(rank, world, port, case, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        W, H, D, K, w_y, m_pool, kind = case
        if kind == "scene":
            L, R, _ = synth.scene(W, H, D, seed=11)
        else:  # unrelated noise: many rows without a single GCP (rule (d))
            L, R = synth.random_pair(W, H, seed=5, levels=256)
        ov = dict(k_scale=K, w_y=w_y, m_pool=m_pool)
        runner = sdist.BandRunner(W, H, D, dist, "cpu", compute=False, **ov)
        b = runner.b
        runner.own_view(0, "L").copy_(torch.from_numpy(L[b.y0:b.y0 + b.rows]))
        runner.own_view(0, "R").copy_(torch.from_numpy(R[b.y0:b.y0 + b.rows]))
        for w in runner.exchange(0):
            w.wait()
        Lb, Rb = runner.Lsub[0].numpy(), runner.Rsub[0].numpy()
        ok_x = np.array_equal(Lb, L[b.sub_y0:b.sub_y0 + b.sub_rows]) and \
            np.array_equal(Rb, R[b.sub_y0:b.sub_y0 + b.sub_rows])
        # band compute (oracle on the sub-image) and its own-row summaries
        p = oracle.params(**ov)
        r = oracle.pipeline(Lb, Rb, D, p, "fixed", stages=("median", "fill", "out"))
        s0, ys0 = b.sub_y0 // K, b.y0 // K
        ys1 = (b.y0 + b.rows) // K if b.y0 + b.rows < H else H // K
        summ_local = _summaries(r["median"])
        runner.summ.fill_(-1)
        runner.summ[ys0:ys1] = torch.from_numpy(summ_local[ys0 - s0:ys1 - s0])
        runner.reduce_summaries()
        summ = runner.summ.numpy()
        # rule (d) from the frame-wide summaries (what stereo_band_finish does)
        fill, out = r["fill"].copy(), r["out"]
        hi = min(ys1 + (1 if K == 2 else 0), H // K)
        patched = [y for y in range(ys0, hi) if summ[y, 0] < 0]
        for y in patched:
            fill[y - s0] = _rule_d_value(summ, y)
        if patched:
            out = fill if K == 1 else oracle.scale_up(fill, Lb, K, p.t_fill)
        mine = out[b.top:b.top + b.rows]
        parts = [None] * world
        dist.all_gather_object(parts, (b.y0, b.rows, mine, ok_x))
        if rank == 0:
            full = oracle.pipeline(L, R, D, p, "fixed", stages=("median", "out"))
            got = np.zeros_like(full["out"])
            for y0, rows, part, _ in parts:
                got[y0:y0 + rows] = part
            ok_summ = np.array_equal(summ, _summaries(full["median"]))
            q.put((all(pt[3] for pt in parts), bool(ok_summ),
                   bool(np.array_equal(got.view(np.uint32), full["out"].view(np.uint32)))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,case", [
    (2, (160, 120, 32, 2, 31, 1, "scene")),
    (3, (96, 150, 24, 1, 7, 1, "scene")),
    (2, (24, 60, 16, 1, 3, 1, "noise")),
    (3, (20, 62, 20, 2, 4, 1, "noise")),
    (3, (10, 90, 16, 2, 1, 1, "noise")),   # rows 26..30 have no GCP: only the global patch is right
    # every pool radius (m_pool = 0 left the band one scaled row short)
    (3, (64, 96, 16, 2, 4, 0, "scene")),
    (3, (64, 96, 16, 2, 4, 2, "scene")),
    (2, (64, 97, 16, 2, 4, 3, "scene")),
    (3, (40, 96, 16, 2, 4, 0, "noise")),
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
    ok_x, ok_summ, ok_out = q.get(timeout=10)
    assert ok_x, "halo exchange delivered wrong rows"
    assert ok_summ, "all-reduced summaries differ from the frame's"
    assert ok_out, "assembled bands differ from the full frame"


def test_band_partition_covers_and_aligns():
    for H, P, K, m in ((992, 8, 2, 1), (991, 3, 2, 1), (375, 4, 1, 1), (1984, 8, 2, 1), (96, 3, 2, 0)):
        p = abi.default_params(k_scale=K, m_pool=m)
        bands = sdist.band_layout(H, P, p)
        assert bands[0].y0 == 0 and bands[-1].y0 + bands[-1].rows == H
        for a, b in zip(bands, bands[1:]):
            assert a.y0 + a.rows == b.y0
        for b in bands:
            assert b.sub_y0 % K == 0 and b.sub_y0 >= 0 and b.sub_y0 + b.sub_rows <= H
            # the cone: w_y + census reach + cross-check/median/Step8 rows, in scaled rows
            # (clipped at the frame's edges)
            assert b.top >= min(b.y0, K * (31 + 2 + 1) + (m if K == 2 else 0))
            assert b.bot >= min(H - b.y0 - b.rows, K * (31 + 2 + 1 + (K == 2)))
    with pytest.raises(abi.StereoError):
        abi.band_rows(10, 8, 0, k_scale=2)
    with pytest.raises(abi.StereoError):  # odd start for K = 2
        abi.band_halo(992, 3, 100, k_scale=2)


def test_halo_sends_cover_every_sub_image():
    p = abi.default_params()
    bands = sdist.band_layout(992, 8, p)
    sends = sdist.halo_sends(bands)
    for b in bands:
        got = set(range(b.y0, b.y0 + b.rows))
        for src, dst, r0, r1 in sends:
            if dst == b.rank:
                got |= set(range(r0, r1))
        assert got == set(range(b.sub_y0, b.sub_y0 + b.sub_rows))
    # neighbours only at c3 / 8 bands (the cone is smaller than a band)
    assert all(abs(s - d) == 1 for s, d, _, _ in sends)


def test_stream_slices_partition():
    for n, P in ((256, 8), (10, 3), (7, 7)):
        got = sorted(i for r in range(P) for i in sdist.stream_slice(n, P, r))
        assert got == list(range(n))


def _c4_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n = 11  # a short stream of the c4 kind (translating scene), split over the ranks
        sl = sdist.stream_slice(n, world, rank)
        mine = synth.stream(48, 32, 8, n, seed=4, idx=sl)
        digests = [(i, int(np.asarray(L, np.int64).sum()), int(np.asarray(R, np.int64).sum()))
                   for i, (L, R) in zip(sl, mine)]
        parts = [None] * world
        dist.all_gather_object(parts, digests)
        if rank == 0:
            full = synth.stream(48, 32, 8, n, seed=4)
            ref = [(i, int(L.astype(np.int64).sum()), int(R.astype(np.int64).sum())) for i, (L, R) in enumerate(full)]
            got = sorted(d for p in parts for d in p)
            q.put(got == ref)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_c4_stream_slices_render_the_whole_stream(world):
    """Config c4: every rank renders only its dist.stream_slice of the frame
    stream (synth.stream(idx=...)); together the ranks hold exactly the frames
    of a whole-stream render, each once."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_c4_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    assert q.get(timeout=10)


@pytest.mark.parametrize("seed", range(20))
def test_band_geometry_random_cases_with_oracle(seed):
    """The library's band partition and halo (stereo_band_rows /
    stereo_band_halo, host functions) on random shapes and parameters: the
    oracle run on every band's sub-image reproduces the whole frame's own
    rows bit for bit, once fill rule (d) is resolved from the frame-wide
    summaries (what stereo_band_finish does)."""
    rng = np.random.default_rng(900 + seed)
    K = int(rng.choice([1, 2]))
    W = int(rng.integers(6, 48))
    H = int(rng.integers(8 * K, 90))
    D = int(rng.integers(1, 12))
    cand = [(dx, dy) for dx in range(-2, 3) for dy in range(-2, 3) if (dx, dy) != (0, 0)]
    pat = [cand[i] for i in rng.choice(len(cand), 6, replace=False)]
    ov = dict(k_scale=K, w_y=int(rng.integers(0, 12)), m_pool=int(rng.integers(0, 4)),
              delta=int(rng.integers(1, 40)), w_x=int(rng.integers(0, 10)), census=pat)
    L, R = synth.random_pair(W, H, seed=seed, levels=int(rng.integers(2, 257)))
    P = int(rng.integers(1, min(5, H // K) + 1))
    p = oracle.params(**ov)
    full = oracle.pipeline(L, R, D, p, "fixed", stages=("median", "out"))
    summ = _summaries(full["median"])
    bands = sdist.band_layout(H, P, abi.default_params(**ov))
    got = np.zeros_like(full["out"])
    for b in bands:
        Lb, Rb = L[b.sub_y0:b.sub_y0 + b.sub_rows], R[b.sub_y0:b.sub_y0 + b.sub_rows]
        r = oracle.pipeline(Lb, Rb, D, p, "fixed", stages=("fill", "out"))
        s0, ys0 = b.sub_y0 // K, b.y0 // K
        ys1 = (b.y0 + b.rows) // K if b.y0 + b.rows < H else H // K
        fill, out = r["fill"].copy(), r["out"]
        hi = min(ys1 + (1 if K == 2 else 0), H // K)
        patched = [y for y in range(ys0, hi) if summ[y, 0] < 0]
        for y in patched:
            fill[y - s0] = _rule_d_value(summ, y)
        if patched:
            out = fill if K == 1 else oracle.scale_up(fill, Lb, K, p.t_fill)
        got[b.y0:b.y0 + b.rows] = out[b.top:b.top + b.rows]
    assert np.array_equal(got.view(np.uint32), full["out"].view(np.uint32)), (W, H, D, P, ov)
