# binning work split per (row, segment) item: 4 lanes vs a warp (BP_BIN_GROUP), 4 M networks
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"; }
for wl in coba4m_p001 coba4m_k1000 coba4m_jit; do for r in 1 2; do
  for g in 4 32 64; do echo -n "$wl group=$g: "; BP_BIN_GROUP=$g run --workload $wl; done
done; done
