# A/B of the fused delivery (BP_FUSED_BIN=0 vs 1) on network workloads
for wl in ${WLS:-coba_lif_jit coba4m_jit coba4m_k1000 coba4m_p001}; do for g in ${GS:-f32}; do for v in 0 1 0 1; do
  echo -n "$wl $g fused=$v: "; BP_FUSED_BIN=$v python bench.py --workload $wl --g $g --steps ${STEPS:-400} --warmup 5 --no-cpu --no-e2e ${BENCH_ARGS} | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2), 'ev/step', d.get('events_per_step'))"
done; done; done
