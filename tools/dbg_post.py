import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle
from paper_2212_00488_b200 import abi, synth
W, H, D, K, w_y, P, seed = (10, 90, 16, 2, 1, 3, 5)
L, R = synth.random_pair(W, H, seed=seed)
st = abi.Stereo(W, H, D, k_scale=K, w_y=w_y)
out = torch.empty((H, W), dtype=torch.float32, device="cuda")
st.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda(), out); torch.cuda.synchronize()
ref = oracle.pipeline(L, R, D, oracle.params(k_scale=K, w_y=w_y), "fixed", stages=("DL","DR","masked","median","fill","out"))
print(list(ref.keys()))
for name, buf in (("DL", abi.BUF_DL), ("DR", abi.BUF_DR), ("masked", abi.BUF_MASKED), ("median", abi.BUF_MEDIAN), ("fill", abi.BUF_FILL)):
    g = st.download(buf)
    r = ref.get(name)
    if r is None: print(name, "no ref"); continue
    bad = np.argwhere(g.reshape(r.shape) != r)
    print(name, g.shape, "mismatches", len(bad), bad[:5])
    if len(bad): print(" got", g.reshape(r.shape)[bad[0][0]], "\n ref", r[bad[0][0]])
