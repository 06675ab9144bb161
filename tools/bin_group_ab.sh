# A/B of the binning kernel's lanes per (row, segment) item (BP_BIN_GROUP)
for wl in coba_lif_jit coba4m_jit coba4m_k1000; do for g in 4 8 32; do echo "== $wl S=$g"; BP_BIN_GROUP=$g python bench.py --workload $wl --steps 200 --warmup 5 --no-cpu --no-e2e | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); r=d['roofline']; print(round(d['ms_per_step']*1e3,2), 'kstep', round(r['avg_launch_us'],2), 'kbin', round(r['bin_kernel']['avg_launch_us'],2))"; done; done
for g in 4 8 32; do echo "== g8 S=$g"; BP_BIN_GROUP=$g python bench.py --emulate-world 8 --steps 200 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; done
