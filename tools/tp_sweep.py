"""Dev tool: multi-stream throughput (frames in flight) at c3 under plan
overrides (STEREO_* knobs read at stereo_create).  Usage:
    python tools/tp_sweep.py "XPASS_WARPS=8,XPASS_SLOTS=2" "YPASS_NB=4" ...
Each argument is one configuration (comma-separated KEY=VALUE, prefix STEREO_
implied); "-" = planner defaults.  Prints fps per configuration and stream count."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2212_00488_b200 import abi, synth  # noqa: E402

W, H, D, K = [int(v) for v in os.environ.get("TP_WHDK", "1436,992,145,2").split(",")]
POOL = 16 if W * H <= 4e6 else 4
frames = [synth.scene(W, H, D, seed=s)[:2] for s in range(POOL)]
Ls = [torch.from_numpy(f[0]).cuda() for f in frames]
Rs = [torch.from_numpy(f[1]).cuda() for f in frames]


def run(cfg, nstreams, n=600):
    for k in list(os.environ):
        if k.startswith("STEREO_"):
            del os.environ[k]
    if cfg != "-":
        for kv in cfg.split(","):
            k, v = kv.split("=")
            os.environ["STEREO_" + k] = v
    hs = [abi.Stereo(W, H, D, k_scale=K) for _ in range(nstreams)]
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    outs = [torch.empty((H, W), dtype=torch.float32, device="cuda") for _ in range(nstreams)]
    info = hs[0].info

    stages = [int(v) for v in os.environ.get("TP_STAGES", "").split(",") if v]

    def go(m):
        for i in range(m):
            j = i % nstreams
            with torch.cuda.stream(ss[j]):
                if stages and i >= nstreams:  # subset of stages on the buffers of a full frame
                    for sid in stages:
                        hs[j].run_stage(sid, Ls[i % POOL], Rs[i % POOL], outs[j], stream=ss[j])
                else:
                    hs[j].compute(Ls[i % POOL], Rs[i % POOL], outs[j])

    go(60)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in ss:
        s.wait_event(e0)
    go(n)
    for s in ss:
        ev = torch.cuda.Event()
        ev.record(s)
        torch.cuda.current_stream().wait_event(ev)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / n
    for h in hs:
        h.close()
    return ms, info


for cfg in sys.argv[1:] or ["-"]:
    for ns in [int(v) for v in os.environ.get("TP_STREAMS", "1,4,6").split(",")]:
        ms, info = run(cfg, ns)
        print(f"{cfg:40s} streams={ns}  {ms*1e3:7.1f} us/frame  {1e3/ms:7.0f} fps", flush=True)
