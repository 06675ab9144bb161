# remote row listing: words per thread 16 (A) / 32 (B) / 8 (C) vs compaction (A + BP_BIN_COMPACT=1)
run() { python bench.py "$@" --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "--emulate-world 8" "--emulate-world 2" "--workload coba4m_jit --emulate-world 8" "--workload coba4m_jit --emulate-world 2"; do
  for r in 1 2; do
    echo -n "$args compact: "; BP_BIN_COMPACT=1 BP_LIB=$PWD/libs_ab/libbp_A.so run $args
    for v in A B C; do echo -n "$args $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so run $args; done
  done
done
