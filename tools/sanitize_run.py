"""One frame of each configuration through the C ABI, for compute-sanitizer
(SURVEY §4 T8): python tools/sanitize_run.py [c1 c2 c3 ...]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_00488_b200 import abi, synth  # noqa: E402

CFG = {"c1": (64, 48, 16, 1), "c2": (450, 375, 64, 1), "c3": (1436, 992, 145, 2),
       "odd": (131, 77, 33, 2), "wide": (2880, 64, 40, 2)}
for name in sys.argv[1:] or ["c1", "c2"]:
    if name == "band":  # one band handle of a 3-band split, plus its summary / finish kernels
        W, H, D = 300, 258, 48
        L, R, _ = synth.scene(W, H, D, seed=3)
        y0, rows = abi.band_rows(H, 3, 1)
        bs = abi.StereoBand(W, H, D, y0, rows)
        Lb = torch.from_numpy(L[bs.sub_y0:bs.sub_y0 + bs.sub_rows].copy()).cuda()
        Rb = torch.from_numpy(R[bs.sub_y0:bs.sub_y0 + bs.sub_rows].copy()).cuda()
        o = torch.empty((rows, W), dtype=torch.float32, device="cuda")
        summ = torch.empty((H // 2, 2), dtype=torch.int32, device="cuda")
        bs.compute(Lb, Rb, o)
        bs.summary(summ)
        bs.finish(summ, Lb, o)
        torch.cuda.synchronize()
        bs.close()
        print(name, "ok", float(o.mean()))
        continue
    W, H, D, K = CFG[name]
    L, R, _ = synth.scene(W, H, D, seed=3)
    st = abi.Stereo(W, H, D, k_scale=K)
    out = torch.empty((H, W), dtype=torch.float32, device="cuda")
    Lt, Rt = torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda()
    st.compute(Lt, Rt, out)
    torch.cuda.synchronize()
    st.close()
    print(name, "ok", float(out.mean()))
