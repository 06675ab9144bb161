"""Per-step kernel times through the initial synchronous burst of the
12.5 M-neuron network (steps 0..N): events per step vs the update and the
binning kernel durations -- does the binning scale with the events?"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2311_05106_b200.network import CobaNetwork  # noqa: E402

torch.cuda.set_device(0)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 12_500_000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 40
net = CobaNetwork(n, conn="jit", fixed=False)
rows = []
for k in range(steps):
    c0 = net.counters()
    net.net.profile_begin(1)
    net.run(1)
    sc, up, _ = net.net.profile_end()
    c1 = net.counters()
    rows.append({"step": k, "spikes": c1[0] - c0[0], "events_binned": c1[1] - c0[1],
                 "k_step_us": up * 1e3, "k_bin_us": sc * 1e3})
    print(json.dumps(rows[-1]), flush=True)
