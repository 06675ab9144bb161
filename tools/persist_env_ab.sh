# persistent k_step for the 4 M networks (977 tiles): default (non-persistent) vs BP_STEP_PERSIST=1
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"; }
for wl in coba4m_jit coba4m_k1000 coba4m_p001; do for r in 1 2; do
  echo -n "$wl default: "; run --workload $wl
  echo -n "$wl persist: "; BP_STEP_PERSIST=1 run --workload $wl
done; done
for g in fix32; do for r in 1 2; do
  echo -n "cfg5 $g default: "; run --g $g
  echo -n "cfg5 $g persist: "; BP_STEP_PERSIST=1 run --g $g
done; done
