"""Multi-GPU plumbing: one process per GPU,
torch.distributed (NCCL over NVLink; gloo in the CPU tests) for the bytes,
the C ABI for everything the method computes.

* **Frame batches** (config c4): frames are independent; every rank computes
  its own contiguous slice of the stream (`stream_slice`), no collective in
  the data path.
* **Row bands** (config c5): rank r owns the band of original rows the
  library's partition gives it (`stereo_band_rows`) and computes it with a
  band handle (`stereo_create_band`).  Per frame this module only MOVES BYTES:

    1. the halo rows of L and R that the band's dependency cone needs
       (`stereo_band_halo`) arrive from the neighbouring ranks in ONE grouped
       P2P step, received straight into the band's preallocated sub-image
       buffer (no temporaries);
    2. `stereo_compute_band` + `stereo_band_summary` (enqueued);
    3. one element-wise MAX all-reduce of the frame-wide int32 [H/K][2] row
       summaries (NCCL, stream-ordered);
    4. `stereo_band_finish` resolves fill rule (d) on the device.

  Nothing synchronises the host.  `BandRunner.run_stream` double-buffers the
  sub-images so that frame i+1's halo exchange (side stream) overlaps frame
  i's compute.
"""
from __future__ import annotations

from dataclasses import dataclass


@dataclass(frozen=True)
class Band:
    rank: int
    y0: int    # own original rows [y0, y0 + rows)
    rows: int
    top: int   # halo rows above / below (the library's dependency cone)
    bot: int

    @property
    def sub_y0(self):  # frame row of the sub-image's first row
        return self.y0 - self.top

    @property
    def sub_rows(self):
        return self.top + self.rows + self.bot


def band_layout(H: int, P: int, params):
    """Every rank's band, from the library's host-side partition and halo
    rules (identical on all ranks: no communication)."""
    from . import abi
    out = []
    for r in range(P):
        y0, rows = abi.band_rows(H, P, r, params)
        top, bot = abi.band_halo(H, y0, rows, params)
        out.append(Band(r, y0, rows, top, bot))
    return out


def halo_sends(bands):
    """(src, dst, row0, row1): frame rows [row0, row1) that src owns and dst's
    sub-image needs."""
    out = []
    for dst in bands:
        for src in bands:
            if src.rank == dst.rank:
                continue
            lo = max(src.y0, dst.sub_y0)
            hi = min(src.y0 + src.rows, dst.sub_y0 + dst.sub_rows)
            if lo < hi:
                out.append((src.rank, dst.rank, lo, hi))
    return out


def stream_slice(n_frames: int, P: int, rank: int):
    """Contiguous slice of a frame stream for frame-batch mode (config c4)."""
    return range(rank * n_frames // P, (rank + 1) * n_frames // P)


class BandRunner:
    """Rank `rank` of a P-way row-band split of W x H frames (P = world size).

    comm_device: where the exchanged bytes live (the GPU for NCCL; the CPU for
    gloo); compute: whether to run the band handle (False in the CPU tests,
    which only exercise the byte movement)."""

    def __init__(self, W, H, D, dist, device, params=None, comm_device=None, compute=True,
                 slots=2, **overrides):
        import torch

        from . import abi
        self.dist = dist
        self.rank, self.P = dist.get_rank(), dist.get_world_size()
        self.p = params if params is not None else abi.default_params(**overrides)
        self.W, self.H, self.D = W, H, D
        self.K = self.p.k_scale
        self.Hs = H // self.K
        self.bands = band_layout(H, self.P, self.p)
        self.b = self.bands[self.rank]
        self.device = torch.device(device)
        self.cdev = torch.device(comm_device) if comm_device is not None else self.device
        b = self.b
        # preallocated, double-buffered sub-images (own rows at [top, top + rows))
        self.Lsub = [torch.zeros((b.sub_rows, W), dtype=torch.uint8, device=self.cdev) for _ in range(slots)]
        self.Rsub = [torch.zeros_like(self.Lsub[0]) for _ in range(slots)]
        if self.cdev != self.device:  # gloo test mode: device copies of the sub-images
            self.Ldev = [torch.empty((b.sub_rows, W), dtype=torch.uint8, device=self.device) for _ in range(slots)]
            self.Rdev = [torch.empty_like(self.Ldev[0]) for _ in range(slots)]
        else:
            self.Ldev, self.Rdev = self.Lsub, self.Rsub
        self.summ = torch.full((self.Hs, 2), -1, dtype=torch.int32, device=self.cdev)
        self.summ_dev = self.summ if self.cdev == self.device else torch.empty(
            (self.Hs, 2), dtype=torch.int32, device=self.device)
        self.sends = [t for t in halo_sends(self.bands) if self.rank in (t[0], t[1])]
        self.st = abi.StereoBand(W, H, D, b.y0, b.rows, params=self.p) if compute else None
        if self.st is not None:
            assert (self.st.top, self.st.bot) == (b.top, b.bot)

    # ---------------------------------------------------------------- bytes
    def own_view(self, slot, img="L"):
        """The own-row region of slot's sub-image (write the frame's own rows here)."""
        t = (self.Lsub if img == "L" else self.Rsub)[slot]
        return t[self.b.top:self.b.top + self.b.rows]

    def exchange(self, slot):
        """Start the one grouped P2P step that fills slot's halo rows; returns
        the work handles (wait() orders the current stream after them)."""
        me = self.b
        ops = []
        for src, dst, r0, r1 in self.sends:
            for buf in (self.Lsub[slot], self.Rsub[slot]):
                if src == self.rank:
                    ops.append(self.dist.P2POp(self.dist.isend, buf[r0 - me.sub_y0:r1 - me.sub_y0], dst))
                else:
                    ops.append(self.dist.P2POp(self.dist.irecv, buf[r0 - me.sub_y0:r1 - me.sub_y0], src))
        return self.dist.batch_isend_irecv(ops) if ops else []

    def reduce_summaries(self):
        """Element-wise MAX over the bands of the frame-wide row summaries
        (one NCCL all-reduce, stream-ordered: no host synchronisation)."""
        if self.summ_dev is not self.summ:
            self.summ.copy_(self.summ_dev)
        self.dist.all_reduce(self.summ, op=self.dist.ReduceOp.MAX)
        if self.summ_dev is not self.summ:
            self.summ_dev.copy_(self.summ)

    # ---------------------------------------------------------------- compute
    def compute(self, slot, out_own, stream=None):
        """compute_band -> summary -> MAX all-reduce -> finish, all enqueued."""
        if self.Ldev is not self.Lsub:
            self.Ldev[slot].copy_(self.Lsub[slot])
            self.Rdev[slot].copy_(self.Rsub[slot])
        self.st.compute(self.Ldev[slot], self.Rdev[slot], out_own, stream=stream)
        self.st.summary(self.summ_dev, stream=stream)
        self.reduce_summaries()
        self.st.finish(self.summ_dev, self.Ldev[slot], out_own, stream=stream)
        return out_own

    def run_frame(self, L_own, R_own, out_own, slot=0):
        """One frame: own rows in, own output rows out (device tensors)."""
        self.own_view(slot, "L").copy_(L_own)
        self.own_view(slot, "R").copy_(R_own)
        for w in self.exchange(slot):
            w.wait()
        return self.compute(slot, out_own)

    def run_stream(self, frames, outs):
        """frames: list of (L_own, R_own); outs: list of f32 [rows][W].  The
        halo exchange of frame i+1 runs on a side stream while frame i
        computes (double-buffered sub-images); no host synchronisation."""
        import torch
        n = len(frames)
        if n == 0:
            return outs
        main = torch.cuda.current_stream(self.device)
        side = torch.cuda.Stream(self.device)
        nslot = len(self.Lsub)
        done = [torch.cuda.Event() for _ in range(nslot)]  # slot free (its frame computed)
        ready = [None] * nslot

        def stage(i):
            s = i % nslot
            side.wait_event(done[s])
            with torch.cuda.stream(side):
                self.own_view(s, "L").copy_(frames[i][0])
                self.own_view(s, "R").copy_(frames[i][1])
                works = self.exchange(s)
                for w in works:
                    w.wait()  # side stream waits for the NCCL work
                ev = torch.cuda.Event()
                ev.record(side)
            ready[s] = ev

        for s in range(nslot):
            done[s].record(main)
        stage(0)
        for i in range(n):
            s = i % nslot
            if i + 1 < n:
                stage(i + 1)
            main.wait_event(ready[s])
            self.compute(s, outs[i])
            done[s].record(main)
        return outs

    def close(self):
        if self.st is not None:
            self.st.close()
            self.st = None
