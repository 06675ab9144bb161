for d in ${DENS:-0.001 0.01 0.1}; do for law in homo uniform; do
python bench.py --workload csrmv --law $law --p ${P:-0.05} --density $d --steps 100 --warmup 10 $EXTRA > gpurun_out/m.log 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/m.log').read().strip().splitlines()[-1]); r=d['roofline']; c=d['config']
print(c['workload'], c['p'], c['density'], 'Gev/s=%.1f'%(d['value']/1e9), 'us=%.1f'%d['call_us']['median'], 'frac=%.3f'%r['frac'])"
done; done
