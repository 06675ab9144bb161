# A/B of two libbp builds on emulated multi-GPU ranks (and the G = 1 step)
for G in 8 2; do for v in A B A B; do
  echo -n "G=$G $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so python bench.py --emulate-world $G --steps 400 --warmup 20 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"
done; done
