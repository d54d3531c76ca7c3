"""Dev tool: throughput of stereo_compute_batch (N contiguous frames per call,
one handle / stream) -- amortises the per-call host path for small frames."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_00488_b200 import abi, synth  # noqa: E402

W, H, D, K = [int(v) for v in os.environ.get("TP_WHDK", "64,48,16,1").split(",")]
NB = int(os.environ.get("TP_BATCH", "64"))
fr = [synth.scene(W, H, max(D, 2), seed=s)[:2] for s in range(NB)]
L = torch.stack([torch.from_numpy(f[0]) for f in fr]).cuda()
R = torch.stack([torch.from_numpy(f[1]) for f in fr]).cuda()
out = torch.empty((NB, H, W), dtype=torch.float32, device="cuda")
st = abi.Stereo(W, H, D, k_scale=K)
for _ in range(3):
    st.compute_batch(L, R, out, NB)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 20
e0.record()
for _ in range(reps):
    st.compute_batch(L, R, out, NB)
e1.record()
torch.cuda.synchronize()
us = e0.elapsed_time(e1) * 1e3 / (reps * NB)
print(f"{W}x{H} D={D} K={K} batch={NB}: {us:.1f} us/frame  {1e6 / us:.0f} fps")
