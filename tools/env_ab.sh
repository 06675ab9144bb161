# A/B of an environment switch: ENVVAR=0 vs 1 on network workloads
V=${ENVVAR:-BP_TILE_LIST}
for wl in ${WLS:-coba_lif_jit}; do for g in ${GS:-f32}; do for v in 0 1 0 1; do
  echo -n "$wl $g $V=$v: "; env $V=$v python bench.py --workload $wl --g $g --steps 400 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"
done; done; done
