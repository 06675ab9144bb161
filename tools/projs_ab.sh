# projection table in shared memory for the binning (B) vs read through L1/L2 (A)
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "" "--workload coba4m_jit" "--workload coba4m_p001" "--emulate-world 8" "--emulate-world 2"; do
  for v in A B A B; do echo -n "[$args] $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so run $args; done
done
