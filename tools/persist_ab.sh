# A/B: persistent k_step (default) vs one block per tile (BP_STEP_PERSIST=0)
for g in f32 fix32 fix64; do for wl in coba_lif_jit coba4m_jit; do for v in 1 0 1 0; do
  echo -n "$wl $g persist=$v: "; BP_STEP_PERSIST=$v python bench.py --workload $wl --g $g --steps 400 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'frac', round(r['frac'],3), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"
done; done; done
