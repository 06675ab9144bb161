#!/bin/bash
# default workload: persistent fused kernel vs two kernels per step, 3 modes
for g in f32 fix32 fix64; do for env in "" "BP_NO_PERSIST=1"; do
  env $env python bench.py --g $g --steps ${STEPS:-2000} --warmup 200 --no-cpu --no-e2e > gpurun_out/pab.log 2>&1 || { tail -3 gpurun_out/pab.log; continue; }
  python - "$g" "${env:-persist}" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/pab.log").read().strip().splitlines()[-1])
print(*sys.argv[1:], "us/step=%.1f" % (d["ms_per_step"] * 1e3), "Gev/s=%.2f" % (d["value"] / 1e9))
PY
done; done
