#!/bin/bash
# per-kernel launch list (gpu__time_duration) of a few CSR calls: homo/uniform x p
for law in homo uniform; do for p in 0.05 0.01; do
  ncu --metrics gpu__time_duration.sum --clock-control none -s 40 -c 12 --csv --log-file gpurun_out/l.csv \
      python bench.py --workload csrmv --law $law --p $p --density 0.1 --steps 10 --warmup 10 > /dev/null 2>&1
  python3 - $law $p <<'PY'
import csv, sys
rows = [r for r in csv.reader(open("gpurun_out/l.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
agg = {}
for r in rows[1:]:
    agg.setdefault(r[ki][:45], []).append(float(r[vi].replace(",", "")))
for k, v in agg.items():
    print(*sys.argv[1:], k.ljust(45), "n=%d" % len(v), "mean=%.2f" % (sum(v) / len(v)))
PY
done; done
