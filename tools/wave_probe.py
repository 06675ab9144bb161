"""k_step time vs network size around the wave boundary (tail effect)."""
import sys
import torch
sys.path.insert(0, ".")
import __graft_entry__ as ge
ge.build_lib()
from paper_2311_05106_b200.network import CobaNetwork
torch.cuda.set_device(0)
for n in [int(x) for x in sys.argv[1:]]:
    net = CobaNetwork(n, conn="jit", fixed=False)
    net.run(300)
    torch.cuda.synchronize()
    net.net.profile_begin(500)
    net.run(500)
    sc, up, k = net.net.profile_end()
    print(f"n={n} tiles={(n + 4095) // 4096} waves={(n + 4095) // 4096 / 592:.2f} "
          f"k_step={up / k * 1e3:.1f} us  per-Mneuron={up / k * 1e3 / n * 1e6:.2f} us  bin={sc / k * 1e3:.1f}")
