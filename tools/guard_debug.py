"""Locate an out-of-bounds write: run the stateless CSR calls one by one with
guarded outputs and report which call touched a guard."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2311_05106_b200 as bp
from paper_2311_05106_b200 import inputs
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from test_gpu_guards import Guards

torch.cuda.set_device(0)
n_rows, n_cols = 3000, 2500
ev = inputs.spike_pattern(n_rows, 0.1, 1)
spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()
ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.05, seed=5, weights="uniform", w0=-1, w1=1)
tip, tix, tdat = (torch.from_numpy(a).cuda() for a in (ip, ix, dat))
for dtype, kind in ((torch.float32, 0), (torch.int64, 1)):
    for data in (tdat, None):
        for mode in ("full", "plan", "small"):
            G = Guards()
            out = G(n_cols, dtype)
            wsb = int(bp.lib().bp_csrmv_workspace_bytes(n_rows, n_cols, kind)) if mode != "small" else bp.workspace_bytes(n_rows)
            ws = G(wsb, torch.uint8)
            plan = bp.csrmv_plan(tip, tix, n_rows, n_cols, dtype, homo=data is None, data=data) if mode == "plan" else None
            bp.event_csrmv(tip, tix, data, 0.5, n_rows, n_cols, spikes, out, ws=ws, plan=plan)
            try:
                G.check(); r = "ok"
            except AssertionError as e:
                r = str(e)
                full, g, n, head, tail = G.bufs[0]
                d = (full[:g] != head).nonzero().flatten()
                r += f" changed head idx {d[:8].tolist()} of {g}"
            print(dtype, "homo" if data is None else "hetero", mode, r, flush=True)
