# k_step tile size: 4096 (B) vs 8192 neurons (C, BP_TILE_SHIFT=13), persistent or not
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"; }
for r in 1 2; do
  echo -n "B: "; BP_LIB=$PWD/libs_ab/libbp_B.so run
  echo -n "C: "; BP_LIB=$PWD/libs_ab/libbp_C.so run
  echo -n "C persist: "; BP_STEP_PERSIST=1 BP_LIB=$PWD/libs_ab/libbp_C.so run
  echo -n "B 4m: "; BP_LIB=$PWD/libs_ab/libbp_B.so run --workload coba4m_jit
  echo -n "C 4m: "; BP_LIB=$PWD/libs_ab/libbp_C.so run --workload coba4m_jit
done
