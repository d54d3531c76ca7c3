"""Band mode through dist.BandRunner on the GPU with a one-rank NCCL group
(the only multi-rank topology one GPU allows): the per-frame path (compute ->
summary -> MAX all-reduce -> finish) and the pipelined stream path run with
torch's CUDA sync-debug mode set to "error", i.e. nothing in them synchronises
the host; the output equals the whole-frame computation bit for bit."""
import os
import socket

import numpy as np
import pytest

from paper_2212_00488_b200 import abi
from paper_2212_00488_b200 import dist as sdist
from paper_2212_00488_b200 import synth

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.fixture
def nccl_one_rank():
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_free_port())
    dev = torch.device("cuda", 0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    yield dist
    dist.destroy_process_group()


def test_band_runner_no_host_sync(nccl_one_rank):
    dist = nccl_one_rank
    W, H, D = 300, 200, 48
    frames = [synth.scene(W, H, D, seed=s)[:2] for s in (1, 2, 3)]
    runner = sdist.BandRunner(W, H, D, dist, "cuda:0")
    b = runner.b
    own = [(torch.from_numpy(L[b.y0:b.y0 + b.rows].copy()).cuda(),
            torch.from_numpy(R[b.y0:b.y0 + b.rows].copy()).cuda()) for L, R in frames]
    outs = [torch.empty((b.rows, W), dtype=torch.float32, device="cuda") for _ in frames]
    runner.run_frame(*own[0], outs[0])  # first call: NCCL communicator set-up
    torch.cuda.synchronize()
    torch.cuda.set_sync_debug_mode("error")
    try:
        runner.run_frame(*own[1], outs[1])
        runner.run_stream(own, outs)
    finally:
        torch.cuda.set_sync_debug_mode("default")
    torch.cuda.synchronize()
    for (L, R), o in zip(frames, outs):
        st = abi.Stereo(W, H, D)
        ref = torch.empty((H, W), dtype=torch.float32, device="cuda")
        st.compute(torch.from_numpy(L).cuda(), torch.from_numpy(R).cuda(), ref)
        torch.cuda.synchronize()
        st.close()
        assert torch.equal(o.view(torch.int32), ref.view(torch.int32))
    runner.close()
