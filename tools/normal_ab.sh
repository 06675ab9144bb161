for p in 0.05 0.01 0.001; do for arm in A B; do
  if [ $arm = B ]; then export BP_JIT_TILED=1; else unset BP_JIT_TILED; fi
  timeout 120 python bench.py --workload jitmv --law normal --p $p --density 0.1 --steps 20 --warmup 5 > gpurun_out/nab.log 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/nab.log').read().strip().splitlines()[-1]); print('$arm', 'normal', $p, 'call_us=%.1f' % d['call_us']['median'])"
done; done
