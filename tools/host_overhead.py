"""Host (CPU) cost of one multi-process step: the two library calls, the
stream switch and the local-slice copy of step_distributed (no collective),
against the GPU step time.  Run on a GPU box: python tools/host_overhead.py"""
import time

import torch

import __graft_entry__ as ge

ge.build_lib()
from paper_2311_05106_b200.network import CobaNetwork  # noqa: E402

torch.cuda.set_device(0)
net = CobaNetwork(12_500_000, conn="jit", fixed=False)
comm = torch.cuda.Stream()
send = torch.empty(net.part.local_words, dtype=torch.int32, device="cuda")
for mode in ("update", "update_overlap"):
    for _ in range(50):
        net.net.scatter()
        net.net.update()
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        net.net.scatter()
        if mode == "update":
            net.net.update()
            send.copy_(net.spikes[:net.part.local_words])
        else:
            net.net.update_overlap(comm)
            with torch.cuda.stream(comm):
                send.copy_(net.spikes[:net.part.local_words])
            torch.cuda.current_stream().wait_stream(comm)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{mode}: host {1e6 * (t1 - t0) / n:.1f} us/step enqueue, "
          f"wall {1e6 * (t2 - t0) / n:.1f} us/step")
