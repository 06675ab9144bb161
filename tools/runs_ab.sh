# run layout (B, default for config 5 f32) vs buckets (A = previous build; and B with BP_RUNS=0)
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round((r.get('bin_kernel') or {}).get('avg_launch_us',0),2))"; }
for r in 1 2; do
  echo -n "A: "; BP_LIB=$PWD/libs_ab/libbp_A.so run
  echo -n "B: "; BP_LIB=$PWD/libs_ab/libbp_B.so run
  echo -n "B runs=0: "; BP_RUNS=0 BP_LIB=$PWD/libs_ab/libbp_B.so run
  echo -n "B fix64 runs=1: "; BP_RUNS=1 BP_LIB=$PWD/libs_ab/libbp_B.so run --g fix64
  echo -n "B fix64 runs=0: "; BP_LIB=$PWD/libs_ab/libbp_B.so run --g fix64
done
