#!/bin/bash
# the large JIT microbench cells (p = 0.05 / 0.01 at 10 % density) x laws
for law in homo uniform normal; do for p in 0.05 0.01; do
  python bench.py --workload jitmv --law $law --p $p --density 0.1 --steps ${STEPS:-30} --warmup 5 ${FIX:+--fix} > gpurun_out/j.log 2>&1 || { tail -2 gpurun_out/j.log; continue; }
  python - $law $p <<'PY'
import json, sys
d = json.loads(open("gpurun_out/j.log").read().strip().splitlines()[-1])
print(*sys.argv[1:], "call_us=%.1f" % d["call_us"]["median"], "Gev/s=%.1f" % (d["value"] / 1e9))
PY
done; done
