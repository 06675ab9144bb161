#!/bin/bash
# A/B of JIT microbench cells across an environment switch: bash tools/jit_env_ab.sh VAR
var=$1
for law in homo uniform; do for p in 0.05 0.01; do for arm in A B; do
  if [ $arm = B ]; then export $var=1; else unset $var; fi
  timeout 120 python bench.py --workload jitmv --law $law --p $p --density 0.1 --steps ${STEPS:-30} --warmup 5 > gpurun_out/jab.log 2>&1 || { tail -2 gpurun_out/jab.log; continue; }
  python - $arm $law $p <<'PY'
import json, sys
d = json.loads(open("gpurun_out/jab.log").read().strip().splitlines()[-1])
print(*sys.argv[1:], "call_us=%.1f" % d["call_us"]["median"], "min=%.1f" % d["call_us"]["min"])
PY
done; done; done
unset $var
