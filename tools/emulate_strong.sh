# per-rank step of the strong-scaling configs, emulated ranks on one GPU
for wl in coba4m_jit hh400k_csr; do
  python bench.py --workload $wl --steps 400 --warmup 20 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$wl G=1', round(d['ms_per_step']*1e3,2))"
  for G in 2 4 8; do
    python bench.py --workload $wl --emulate-world $G --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print('$wl G=$G', round(d['ms_per_step']*1e3,2))"
  done
done
