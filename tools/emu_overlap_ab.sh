# emulated weak-scaling rank: stand-in exchange serial (A) vs overlapping the local binning (B)
for G in 2 8; do for r in 1 2; do
  echo -n "G=$G serial: "; python bench.py --emulate-world $G --emu-serial --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2), round(d['config']['events_per_step']))"
  echo -n "G=$G overlap: "; python bench.py --emulate-world $G --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2), round(d['config']['events_per_step']))"
done; done
for wl in coba4m_jit hh400k_csr; do for G in 2 8; do
  echo -n "$wl G=$G serial: "; python bench.py --workload $wl --emulate-world $G --emu-serial --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"
  echo -n "$wl G=$G overlap: "; python bench.py --workload $wl --emulate-world $G --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"
done; done
