"""Quick per-stage device timing at BASELINE config c3 (dev tool, not the bench).
QT_BATCH=n: n frames per launch sequence (stereo_create_batch), as bench.py runs."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_00488_b200 import abi, synth

W, H, D = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1436, 992, 145))]
K = int(sys.argv[4]) if len(sys.argv) > 4 else 2
NB = int(os.environ.get("QT_BATCH", "1"))
fr = [synth.scene(W, H, D, seed=s)[:2] for s in range(NB)]
st = abi.Stereo(W, H, D, k_scale=K, max_frames=NB)
Lt = torch.from_numpy(np.stack([f[0] for f in fr])).cuda()
Rt = torch.from_numpy(np.stack([f[1] for f in fr])).cuda()
out = torch.empty((NB, H, W), dtype=torch.float32, device="cuda")
run = lambda: st.compute_batch(Lt, Rt, out, NB)
for _ in range(10): run()
torch.cuda.synchronize()
n = max(200 // NB, 20)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): run()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / (n * NB)
st.set_timing(True)
for _ in range(n): run()
t, nf = st.stage_times_ms()
i = st.info
print(f"{W}x{H} D={D} K={K} ({NB} frame(s) per launch): {ms*1e3:.1f} us/frame  {1e3/ms:.0f} fps")
vol = i.Ds * i.Hs * i.Ws * 4 * 2
for k, v in t.items():
    us = v / nf * 1e3
    extra = ""
    if us <= 0:
        continue
    if k == "XPASS": extra = f"  write {vol/1e6:.0f} MB -> {vol/us/1e3:.0f} GB/s"
    if k == "YPASS": extra = f"  read {vol/1e6:.0f} MB -> {vol/us/1e3:.0f} GB/s"
    print(f"  {k:6s} {us:8.1f} us{extra}")
