"""The N > 1 host loop on one GPU (NCCL, world size 1, 12.5 M neurons, f32):
eager step_distributed vs the captured CUDA graph vs the single-process
library loop, device-timed with CUDA events.
Run on a GPU box: PYTHONPATH=. python tools/dist_loop_timing.py"""
import os

import torch
import torch.distributed as dist

import __graft_entry__ as ge

ge.build_lib()
from paper_2311_05106_b200.network import CobaNetwork  # noqa: E402

os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
os.environ.setdefault("MASTER_PORT", "29561")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
K = 2000


def timed(fn):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) * 1e3 / K


net = CobaNetwork(12_500_000, conn="jit", fixed=False, world=1)
for _ in range(200):
    net.step_distributed()
print("eager step_distributed (overlap): %.1f us/step" %
      timed(lambda: [net.step_distributed() for _ in range(K)]))
print("eager step_distributed (no overlap): %.1f us/step" %
      timed(lambda: [net.step_distributed(overlap=False) for _ in range(K)]))
g, period = net.capture()
g.replay()
print("captured graph of %d steps: %.1f us/step" %
      (period, timed(lambda: [g.replay() for _ in range(K // period)])))
print("library loop (bp_network_step): %.1f us/step" % timed(lambda: net.run(K)))
dist.destroy_process_group()
