"""Step-by-step GPU vs oracle comparison of a small COBA network (debug aid)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import oracle  # noqa: E402
from paper_2311_05106_b200 import inputs  # noqa: E402
from paper_2311_05106_b200.network import SEED_E, SEED_I, CobaNetwork  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4000
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
net = CobaNetwork(n, conn="jit", fixed=True)
n_exc = n * 4 // 5
K = oracle.conn_len(80.0 / n)
pe = oracle.Projection(0, n_exc, jit=oracle.JitSpec(SEED_E, K, n, oracle.LAW_HOMO, 0.6))
pi = oracle.Projection(n_exc, n - n_exc, jit=oracle.JitSpec(SEED_I, K, n, oracle.LAW_HOMO, 6.7))
st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
          ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
for k in range(steps):
    net.run(1)
    r = oracle.run_network("lif", oracle.lif_params(), st, pe, pi, 1)
    gv = net.state["v"].cpu().numpy()
    ge = net.state["g_e"].cpu().numpy()
    gi = net.state["g_i"].cpu().numpy()
    sp = inputs.unpack_bits(net.spikes.cpu().numpy().view(np.uint32), n)
    bad_v = np.nonzero(gv.view(np.uint32) != st["v"].view(np.uint32))[0]
    bad_e = np.nonzero(ge != st["g_e"])[0]
    bad_i = np.nonzero(gi != st["g_i"])[0]
    bad_s = np.nonzero(sp != r[0])[0]
    if len(bad_v) or len(bad_e) or len(bad_i) or len(bad_s):
        print(f"step {k}: spikes gpu {sp.sum()} oracle {r[0].sum()}; bad v {len(bad_v)} "
              f"ge {len(bad_e)} gi {len(bad_i)} spikes {len(bad_s)}")
        for name, bad, a, b in (("ge", bad_e, ge, st["g_e"]), ("gi", bad_i, gi, st["g_i"]),
                                ("v", bad_v, gv, st["v"])):
            for j in bad[:5]:
                print(f"  {name}[{j}] gpu {a[j]} oracle {b[j]}  ratio {a[j] / max(b[j], 1e-30)}")
        print("  bad spike ids", bad_s[:10])
        break
else:
    print(f"all {steps} steps identical; total spikes {net.counters()}")
