#!/bin/bash
# non-event JIT mv cells (NEXT 1): 100k x 100k, p x non-zero density, 3 laws
for law in homo uniform normal; do for p in 0.05 0.01; do for d in 1.0 0.1; do
  python bench.py --workload jitmv_vec --law $law --p $p --density $d --steps ${STEPS:-20} --warmup 3 ${FIX:+--fix} > gpurun_out/v.log 2>&1 || { tail -2 gpurun_out/v.log; continue; }
  python - $law $p $d <<'PY'
import json, sys
d = json.loads(open("gpurun_out/v.log").read().strip().splitlines()[-1])
print(*sys.argv[1:], "call_us=%.1f" % d["call_us"]["median"], "Gev/s=%.1f" % (d["value"] / 1e9),
      "frac=%.3f" % d["roofline"]["frac"])
PY
  cat gpurun_out/v.log >> gpurun_out/mv_cells.jsonl
done; done; done
