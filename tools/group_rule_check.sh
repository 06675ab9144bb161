# the lanes-per-item rule as chosen by the library (no override) on the emulated ranks
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "--emulate-world 8" "--emulate-world 2" "--workload coba4m_jit --emulate-world 8" "--workload coba4m_jit --emulate-world 4"; do
  echo -n "[$args] default: "; run $args
done
