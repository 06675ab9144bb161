for mode in "" "--f32"; do for keep in 0 60 91 110; do
  BP_L2_KEEP_MB=$keep python bench.py --steps 2000 --warmup 200 --no-cpu --no-e2e $mode > gpurun_out/sw_${keep}${mode}.log 2>&1
  python -c "
import json,sys; d=json.loads(open('gpurun_out/sw_${keep}${mode}.log').read().strip().splitlines()[-1]); r=d['roofline']
print('keep=$keep mode=$mode', 'us/step=%.1f'%(d['ms_per_step']*1e3), 'Gev/s=%.2f'%(d['value']/1e9), 'lif_us=%.1f'%r['avg_launch_us'], 'scat_us=%.1f'%r['scatter_avg_us'], 'ev/step=%d'%d['events_per_step'])"
done; done
