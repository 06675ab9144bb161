# the same preferred shared-memory carveout for the step and binning kernels
for c in "" 72 100 60; do
  echo -n "carveout=$c: "; BP_CARVEOUT=$c python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"
done
