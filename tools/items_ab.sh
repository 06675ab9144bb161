# item-path binning A (HEAD) vs B (working tree): config 3, Fig S3B/S3C, emulated weak-scaling ranks
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "--workload coba4m_jit" "--workload coba4m_k1000" "--workload coba4m_p001" "--emulate-world 8" "--emulate-world 2" "--workload coba4m_jit --emulate-world 8"; do
  for v in A B A B; do echo -n "$args $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so run $args; done
done
