# A/B: dense HH update kernel delivering its own spikes (BP_HH_FUSED=1, default) vs the binning launch (0)
run() { python bench.py --workload hh400k_csr "$@" --steps 2000 --warmup 20 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2), 'ev/step', round(d['config'].get('events', d['config'].get('events_per_step', 0)) or 0))"; }
for r in 1 2; do for f in 0 1; do
  echo -n "G=1 fused=$f: "; BP_HH_FUSED=$f run
  for G in 2 8; do echo -n "G=$G fused=$f: "; BP_HH_FUSED=$f run --emulate-world $G; done
done; done
