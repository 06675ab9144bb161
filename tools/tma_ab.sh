#!/bin/bash
# A/B of the network step kernels: BP_STEP_TMA=0 (k_step) vs 1 (k_step_tma)
for g in f32 fix32 fix64; do for v in 0 1; do
  BP_STEP_TMA=$v timeout 200 python bench.py --g $g --steps 2000 --warmup 200 --no-cpu --no-e2e > gpurun_out/tab.log 2>&1 || { tail -3 gpurun_out/tab.log; continue; }
  python - $g $v <<'PY'
import json, sys
d = json.loads(open("gpurun_out/tab.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(*sys.argv[1:], "us/step=%.1f" % (d["ms_per_step"] * 1e3), "kern=%.1f" % r["avg_launch_us"], "bin=%.1f" % r["bin_kernel_avg_us"], "spikes=%d" % d["config"]["spikes"])
PY
done; done
