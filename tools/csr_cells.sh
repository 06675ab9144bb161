#!/bin/bash
# the three HBM-bound config-2 CSR cells (p=0.05 d=10%, p=0.01 d=10%) x weights x output kind
python -c "import __graft_entry__ as g; g.build_lib()"
for law in homo uniform; do for p in 0.05 0.01; do for fix in "" "--fix"; do
  python bench.py --workload csrmv --law $law --p $p --density 0.1 --steps ${STEPS:-50} --warmup 10 $fix > gpurun_out/c.log 2>&1 || { tail -3 gpurun_out/c.log; continue; }
  python - $law $p "$fix" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/c.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(*sys.argv[1:], "Gev/s=%.1f" % (d["value"] / 1e9), "call_us=%.1f" % d["call_us"]["median"],
      "frac=%.3f" % r["frac"], r["bound"])
PY
  cat gpurun_out/c.log >> gpurun_out/csr_cells.jsonl
done; done; done
