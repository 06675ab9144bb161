#!/bin/bash
# A/B of CSR microbench cells across an environment switch:
#   bash tools/csr_env_ab.sh VAR   (runs every cell with VAR unset, then VAR=1)
var=$1
for law in homo uniform; do for p in 0.05 0.01 0.001; do for arm in A B; do
  if [ $arm = B ]; then export $var=1; else unset $var; fi
  timeout 120 python bench.py --workload csrmv --law $law --p $p --density 0.1 --steps ${STEPS:-50} --warmup 10 ${FIX:+--fix} > gpurun_out/cab.log 2>&1 || { tail -2 gpurun_out/cab.log; continue; }
  python - $arm $law $p <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cab.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(*sys.argv[1:], "call_us=%.1f" % d["call_us"]["median"], "min=%.1f" % d["call_us"]["min"], "frac=%.3f" % r["frac"])
PY
done; done; done
unset $var
