# lanes per item for rows with ~10 events per segment: 2 / 4 / 8
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for args in "--workload coba4m_jit" "--emulate-world 8" "--emulate-world 2" "--workload coba4m_jit --emulate-world 8"; do
  for r in 1 2; do for g in 2 4; do echo -n "[$args] lanes=$g: "; BP_BIN_GROUP=$g run $args; done; done
done
