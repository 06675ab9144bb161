#!/bin/bash
# NEXT 4: gap-sampler cost (uniform U[1,K] vs geometric Geo(p)) on the
# config-2 shape: row regeneration alone (jitrows) and the event scatter.
out=gpurun_out/geo_cells.jsonl; : > $out
for p in 0.05 0.01 0.001; do for gap in uniform geometric; do
  python bench.py --workload jitrows --gap $gap --p $p --steps ${STEPS:-30} --warmup 5 2>/dev/null | grep '^{' >> $out
done; done
for law in homo uniform; do for p in 0.05 0.01; do for gap in uniform geometric; do
  python bench.py --workload jitmv --law $law --gap $gap --p $p --density 0.1 --steps ${STEPS:-30} --warmup 5 2>/dev/null | grep '^{' >> $out
done; done; done
python - <<'PY'
import json
for l in open("gpurun_out/geo_cells.jsonl"):
    d = json.loads(l); c = d["config"]
    print(c["workload"], c["p"], "call_us=%.1f" % d["call_us"]["median"], "Gev/s=%.2f" % (d["value"] / 1e9))
PY
