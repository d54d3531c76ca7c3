"""Quick per-stage device timing at BASELINE config c3 (dev tool, not the bench)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2212_00488_b200 import abi, synth

W, H, D = [int(v) for v in (sys.argv[1:4] if len(sys.argv) > 3 else (1436, 992, 145))]
K = int(sys.argv[4]) if len(sys.argv) > 4 else 2
L, R, _ = synth.scene(W, H, D, seed=0)
st = abi.Stereo(W, H, D, k_scale=K)
Lt, Rt = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
for _ in range(10): st.compute(Lt, Rt, out)
torch.cuda.synchronize()
n = 200
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(n): st.compute(Lt, Rt, out)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
st.set_timing(True)
for _ in range(n): st.compute(Lt, Rt, out)
t, nf = st.stage_times_ms()
i = st.info
print(f"{W}x{H} D={D} K={K}: {ms*1e3:.1f} us/frame  {1e3/ms:.0f} fps")
vol = i.Ds * i.Hs * i.Ws * 4 * 2
for k, v in t.items():
    us = v / nf * 1e3
    extra = ""
    if k == "XPASS": extra = f"  write {vol/1e6:.0f} MB -> {vol/us/1e3:.0f} GB/s"
    if k == "YPASS": extra = f"  read {vol/1e6:.0f} MB -> {vol/us/1e3:.0f} GB/s"
    print(f"  {k:6s} {us:8.1f} us{extra}")
