import os, sys, numpy as np, torch
sys.path.insert(0, "/root/repo")
import paper_2311_05106_b200 as bp
from paper_2311_05106_b200 import inputs
n_rows, n_cols, p, law, density = 50, 70, 0.2, "homo", 0.5
ip, ix, dat = inputs.random_csr(n_rows, n_cols, p, seed=n_rows + n_cols, weights=law)
ev = inputs.spike_pattern(n_rows, density, seed=3)
spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()
tip, tix = torch.from_numpy(ip).cuda(), torch.from_numpy(ix).cuda()
for kind in (torch.int64, torch.float32):
    out = torch.zeros(n_cols, dtype=kind, device="cuda")
    bp.event_csrmv(tip, tix, None, 0.6, n_rows, n_cols, spikes, out)
    torch.cuda.synchronize()
    print(kind, out[:8].tolist())
print("ok")
