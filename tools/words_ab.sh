# A/B: remote binning with its own row listing (k_bin_sorted<true>, default)
# vs compaction launch + list binning (BP_BIN_COMPACT=1), emulated ranks
for G in ${GS:-2 8}; do for v in A B A B; do
  if [ $v = A ]; then export BP_BIN_COMPACT=1; else unset BP_BIN_COMPACT; fi
  echo -n "G=$G $v: "; python bench.py --emulate-world $G --steps 400 --warmup 20 ${BENCH_ARGS} | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2), 'ev/step', d['config'].get('events_per_step'))"
done; done
unset BP_BIN_COMPACT
for wl in coba4m_jit hh400k_csr; do for G in 2 8; do for v in A B; do
  if [ $v = A ]; then export BP_BIN_COMPACT=1; else unset BP_BIN_COMPACT; fi
  echo -n "$wl G=$G $v: "; python bench.py --workload $wl --emulate-world $G --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"
done; done; done
