# config 2 microbenchmark cells (100k x 100k)
for w in ${WORKLOADS:-csrmv jitmv}; do for law in homo uniform normal; do for p in 0.001 0.01 0.05; do for d in 0.001 0.01 0.1; do
  if [ $w = csrmv ] && [ $law = normal ]; then continue; fi
  python bench.py --workload $w --law $law --p $p --density $d --steps ${STEPS:-100} --warmup 10 > gpurun_out/m.log 2>&1 || { tail -3 gpurun_out/m.log; continue; }
  python - $w $law $p $d <<'PY'
import json, sys
d = json.loads(open("gpurun_out/m.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(*sys.argv[1:], "Gev/s=%.1f" % (d["value"] / 1e9), "call_us=%.1f" % d["call_us"]["median"],
      "frac=%.3f" % r["frac"], r["bound"], "ev/call=%d" % d["config"]["events_per_call"])
PY
  cat gpurun_out/m.log >> gpurun_out/micro_all.jsonl
done; done; done; done
