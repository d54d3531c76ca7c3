"""Dev tool: frames/s of stereo_compute_batch with NS handles (one per stream)
of batch capacity NB, frames round-robin over the streams, device-resident.

    python tools/tp_batch.py c1 "1x1,1x64,2x64,4x1" [frames]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2212_00488_b200 import abi, synth  # noqa: E402

CFG = {"c1": (64, 48, 16, 1), "c2": (450, 375, 64, 1), "c3": (1436, 992, 145, 2),
       "c5": (2872, 1984, 290, 2), "vintage": (1444, 960, 380, 2), "pipes": (1482, 994, 128, 2),
       "k1": (1436, 992, 145, 1)}


def run(name, combos, nframes=None):
    W, H, D, K = CFG[name]
    pool = 16
    fr = [synth.scene(W, H, D, seed=i)[:2] for i in range(min(pool, 4))]
    Lp = torch.from_numpy(np.stack([fr[i % len(fr)][0] for i in range(pool)])).cuda()
    Rp = torch.from_numpy(np.stack([fr[i % len(fr)][1] for i in range(pool)])).cuda()
    res = {}
    for c in combos:
        ns, nb = (int(v) for v in c.split("x"))
        hs = [abi.Stereo(W, H, D, k_scale=K, max_frames=nb) for _ in range(ns)]
        ss = [torch.cuda.Stream() for _ in range(ns)]
        nb_pool = min(nb, pool)
        reps = max(1, nb // pool)
        Lb = Lp[:nb_pool].repeat(reps, 1, 1)[:nb].contiguous() if nb > 1 else Lp[:1]
        Rb = Rp[:nb_pool].repeat(reps, 1, 1)[:nb].contiguous() if nb > 1 else Rp[:1]
        outs = [torch.empty((nb, H, W), dtype=torch.float32, device="cuda") for _ in range(ns)]
        n = nframes or max(64, 8 * nb * ns)
        steps = max(ns, n // nb)

        def go(k):
            for i in range(k):
                j = i % ns
                hs[j].compute_batch(Lb, Rb, outs[j], nb, stream=ss[j])

        go(2 * ns)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        main = torch.cuda.current_stream()
        e0.record(main)
        for s in ss:
            s.wait_stream(main)
        go(steps)
        for s in ss:
            main.wait_stream(s)
        e1.record(main)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
        res[c] = steps * nb / (ms / 1e3)
        print(f"{name} streams x batch {c}: {res[c]:.0f} fps ({ms / (steps * nb) * 1e3:.1f} us/frame)", flush=True)
        for h in hs:
            h.close()
    return res


if __name__ == "__main__":
    run(sys.argv[1], sys.argv[2].split(","), int(sys.argv[3]) if len(sys.argv) > 3 else None)
