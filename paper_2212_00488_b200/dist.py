"""Multi-GPU drivers: one process per GPU.

* **Frame batches** (config c4): frames are independent; every rank computes
  its own slice of the stream (`stream_slice`), no collective in the data path.
* **Row bands** (config c5): rank r owns scaled rows [ys0, ys1) of one frame.
  A band is computed by running the unchanged pipeline on a sub-image whose
  halo covers the dependency cone of the band's own rows:

      SU reads fill row y+1 (K=2) | median reads masked rows y-1..y+1
      | WTA reads CA_x rows y-w_y..y+w_y and the y arms of row y (image rows
      y-w_y..y+w_y) | census reads image rows +-max|dy| | Eq. 2 reads
      original rows 2y-m..2y+m

  i.e. `up = w_y + cy + 1` scaled rows above and `down = up + (K == 2)` below,
  plus m original rows, the sub-image starting on an even original row so that
  the scaled grids coincide.  The halo rows of L_org and R_org are exchanged
  with the neighbouring ranks in ONE grouped P2P step (NCCL send/recv over
  NVLink; gloo in the CPU tests).  Only fill rule (d) (a row without any valid
  pixel takes the nearest valid value in raster order) can need rows of other
  bands: the per-row summaries are all-gathered and the (rare) affected rows
  are patched with `stereo_patch_rows`.  Band output == full-frame output, bit
  for bit (tests/test_gpu_bands.py, tests/test_dist_gloo.py).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Band:
    rank: int
    ys0: int  # own scaled rows [ys0, ys1)
    ys1: int
    r0: int   # sub-image original rows [r0, r1)
    r1: int
    o0: int   # own output (original) rows [o0, o1)
    o1: int

    @property
    def rows(self):
        return self.r1 - self.r0


def band_plan(H: int, P: int, K: int = 2, w_y: int = 31, m_pool: int = 1, cy: int = 2):
    """Partition the Hs = H // K scaled rows into P bands (as even as possible)."""
    Hs = H // K
    if P < 1 or P > Hs:
        raise ValueError(f"cannot split {Hs} scaled rows into {P} bands")
    up = w_y + cy + 1
    down = up + (1 if K == 2 else 0)
    bands = []
    for r in range(P):
        ys0, ys1 = r * Hs // P, (r + 1) * Hs // P
        if K == 2:
            r0 = max(0, 2 * (ys0 - up) - m_pool)
            r0 -= r0 & 1
            r1 = min(H, 2 * (ys1 + down - 1) + m_pool + 1)
            o0, o1 = 2 * ys0, (2 * ys1 if ys1 < Hs else H)
        else:
            r0, r1 = max(0, ys0 - up), min(H, ys1 + down)
            o0, o1 = ys0, (ys1 if ys1 < Hs else H)
        bands.append(Band(r, ys0, ys1, r0, r1, o0, o1))
    return bands


def owned_rows(b: Band, H: int, K: int):
    """Original rows a rank holds before the exchange (its own output rows,
    which for K=2 include the odd-H extra row of the last band)."""
    return b.o0, b.o1


def halo_sends(bands, H, K):
    """List of (src_rank, dst_rank, row0, row1): original rows src owns that dst
    needs for its sub-image."""
    out = []
    for dst in bands:
        for src in bands:
            if src.rank == dst.rank:
                continue
            a0, a1 = owned_rows(src, H, K)
            lo, hi = max(a0, dst.r0), min(a1, dst.r1)
            if lo < hi:
                out.append((src.rank, dst.rank, lo, hi))
    return out


def exchange_halos(L_own, R_own, bands, rank, H, K, dist, device=None):
    """Build this rank's sub-image [r0, r1) of L and R from its own rows plus
    the neighbours' rows, in one grouped P2P exchange.

    L_own, R_own: torch u8 [own rows][W] on the communication device (CUDA for
    NCCL, CPU for gloo).  Returns (L_band, R_band) torch u8 [rows][W].
    """
    import torch
    me = bands[rank]
    W = L_own.shape[1]
    a0, a1 = owned_rows(me, H, K)
    Lb = torch.empty((me.rows, W), dtype=L_own.dtype, device=L_own.device)
    Rb = torch.empty_like(Lb)
    lo, hi = max(a0, me.r0), min(a1, me.r1)
    Lb[lo - me.r0:hi - me.r0] = L_own[lo - a0:hi - a0]
    Rb[lo - me.r0:hi - me.r0] = R_own[lo - a0:hi - a0]
    ops, recv = [], []
    for src, dst, r0, r1 in halo_sends(bands, H, K):
        if src == rank:
            for img in (L_own, R_own):
                ops.append(dist.P2POp(dist.isend, img[r0 - a0:r1 - a0].contiguous(), dst))
        elif dst == rank:
            for tgt in (Lb, Rb):
                buf = torch.empty((r1 - r0, W), dtype=L_own.dtype, device=L_own.device)
                ops.append(dist.P2POp(dist.irecv, buf, src))
                recv.append((tgt, r0, buf))
    if ops:
        for req in dist.batch_isend_irecv(ops):
            req.wait()
    for tgt, r0, buf in recv:
        tgt[r0 - me.r0:r0 - me.r0 + buf.shape[0]] = buf
    return Lb, Rb


def rule_d_patches(summ_global, b: Band, K: int, band_rows_scaled: int):
    """Global fill rule (d) for this band.

    summ_global: int [3][Hs] over the whole frame: has_valid, first value, last
    value of every scaled row (all-gathered from each band's own rows).
    Returns (rows_local, values) for every all-invalid row the band's output
    depends on (own rows, plus row ys1 for the scale-up, K = 2)."""
    has, first, last = summ_global
    Hs = has.shape[0]
    rows, vals = [], []
    hi = min(b.ys1 + (1 if K == 2 else 0), Hs)
    s0 = b.r0 // K  # first scaled row of the sub-image
    for y in range(b.ys0, hi):
        if has[y]:
            continue
        v = 0.0
        above = np.nonzero(has[:y])[0]
        if len(above):
            v = float(last[above[-1]])
        else:
            below = np.nonzero(has[y + 1:])[0]
            if len(below):
                v = float(first[y + 1 + below[0]])
        if 0 <= y - s0 < band_rows_scaled:
            rows.append(y - s0)
            vals.append(v)
    return np.array(rows, np.int32), np.array(vals, np.float32)


def gather_row_summaries(local_rows, b: Band, Hs: int, dist, device):
    """all_gather each band's own-row summaries -> int [3][Hs]."""
    import torch
    P = dist.get_world_size()
    own = torch.tensor(local_rows, dtype=torch.int64, device=device)  # [3][own]
    n_max = max(1, -(-Hs // P) + 1)
    pad = torch.full((3, n_max), -2, dtype=torch.int64, device=device)
    pad[:, :own.shape[1]] = own
    meta = torch.tensor([b.ys0, b.ys1], dtype=torch.int64, device=device)
    pads = [torch.empty_like(pad) for _ in range(P)]
    metas = [torch.empty_like(meta) for _ in range(P)]
    dist.all_gather(pads, pad)
    dist.all_gather(metas, meta)
    out = np.zeros((3, Hs), np.int64)
    for pd, mt in zip(pads, metas):
        y0, y1 = (int(v) for v in mt.cpu())
        out[:, y0:y1] = pd[:, :y1 - y0].cpu().numpy()
    return out


class BandStereo:
    """Per-rank band computation on the GPU through the C ABI."""

    def __init__(self, W, H, D, P, rank, params=None, **overrides):
        from . import abi
        self.abi = abi
        self.p = params if params is not None else abi.default_params(**overrides)
        self.K = self.p.k_scale
        cy = max(abs(int(v)) for v in self.p.census_dy)
        self.bands = band_plan(H, P, self.K, self.p.w_y, self.p.m_pool, cy)
        self.b = self.bands[rank]
        self.W, self.H, self.D, self.rank = W, H, D, rank
        self.st = abi.Stereo(W, self.b.rows, D, params=self.p)

    def compute(self, L_band, R_band, out_band, stream=None):
        """Sub-image in, sub-image disparity out (device tensors)."""
        self.st.compute(L_band, R_band, out_band, stream=stream)

    def local_summaries(self):
        """has_valid / first / last value of the band's OWN scaled rows."""
        rows = self.st.download(self.abi.BUF_ROWS)  # [4][Hs_band]
        s0 = self.b.r0 // self.K
        sl = slice(self.b.ys0 - s0, self.b.ys1 - s0)
        return np.stack([(rows[1, sl] >= 0).astype(np.int64), rows[2, sl], rows[3, sl]])

    def needs_patch_local(self):
        """True if a row the band's output reads has no valid pixel."""
        rows = self.st.download(self.abi.BUF_ROWS)
        s0 = self.b.r0 // self.K
        hi = min(self.b.ys1 + (1 if self.K == 2 else 0), self.H // self.K) - s0
        return bool((rows[1, self.b.ys0 - s0:hi] < 0).any())

    def patch(self, summ_global, L_band, out_band, stream=None):
        rows, vals = rule_d_patches(summ_global, self.b, self.K, self.st.info.Hs)
        if len(rows):
            self.st.patch_rows(rows, vals, L_band, out_band, stream=stream)
        return len(rows)

    def own_slice(self):
        return slice(self.b.o0 - self.b.r0, self.b.o1 - self.b.r0)

    def close(self):
        self.st.close()


def run_band_frame(L_own, R_own, W, H, D, dist, device, stereo: BandStereo | None = None,
                   **overrides):
    """One frame in band mode on this rank: exchange halos, compute the band,
    fix rule (d) globally if any band needs it; returns this rank's own output
    rows (f32 [o1-o0][W], device) and the BandStereo (reusable).  The
    exchange runs on L_own's device (CUDA for NCCL; CPU for gloo, whose bands
    are then copied to `device`)."""
    import torch
    rank, P = dist.get_rank(), dist.get_world_size()
    bs = stereo or BandStereo(W, H, D, P, rank, **overrides)
    cdev = L_own.device
    Lb, Rb = exchange_halos(L_own, R_own, bs.bands, rank, H, bs.K, dist)
    if Lb.device != torch.device(device):
        Lb, Rb = Lb.to(device), Rb.to(device)
    out = torch.empty((bs.b.rows, W), dtype=torch.float32, device=device)
    bs.compute(Lb, Rb, out)
    torch.cuda.synchronize(device)
    flag = torch.tensor([1 if bs.needs_patch_local() else 0], device=cdev)
    dist.all_reduce(flag, op=dist.ReduceOp.MAX)
    if int(flag.item()):
        summ = gather_row_summaries(bs.local_summaries(), bs.b, H // bs.K, dist, cdev)
        bs.patch(summ, Lb, out)
    return out[bs.own_slice()], bs


def stream_slice(n_frames: int, P: int, rank: int):
    """Contiguous slice of a frame stream for frame-batch mode."""
    return range(rank * n_frames // P, (rank + 1) * n_frames // P)
