# A/B/C of three libbp builds (libs_ab/libbp_{A,B,C}.so) on network workloads
for wl in ${WLS:-coba_lif_jit coba4m_jit}; do for g in ${GS:-f32 fix64}; do for v in A B C A B C; do
  echo -n "$wl $g $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so python bench.py --workload $wl --g $g --steps 400 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"
done; done; done
