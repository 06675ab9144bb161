#!/bin/bash
# A/B of CSR microbench cells across library builds: bash tools/csr_ab.sh libA.so libB.so ...
for lib in "$@"; do for law in homo uniform; do for p in 0.05 0.01; do
  BP_LIB=$PWD/paper_2311_05106_b200/$lib python bench.py --workload csrmv --law $law --p $p --density 0.1 --steps 30 --warmup 10 ${FIX:+--fix} > gpurun_out/cab.log 2>&1 || { tail -2 gpurun_out/cab.log; continue; }
  python - $lib $law $p <<'PY'
import json, sys
d = json.loads(open("gpurun_out/cab.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(*sys.argv[1:], "call_us=%.1f" % d["call_us"]["median"], "frac=%.3f" % r["frac"])
PY
done; done; done
