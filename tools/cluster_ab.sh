# binning in cluster pairs (BP_BIN_CLUSTER=1) vs single CTAs (0)
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "" "--emulate-world 8" "--emulate-world 2" "--g fix64"; do
  for v in 0 1 0 1; do echo -n "[$args] cluster=$v: "; BP_BIN_CLUSTER=$v run $args; done
done
