# A/B of two libbp builds on the config-2 JIT cells
for cell in "--law homo --p 0.05 --density 0.1" "--law homo --p 0.01 --density 0.1" "--law homo --p 0.05 --density 0.01" "--law uniform --p 0.05 --density 0.1"; do for v in A B A B; do
  echo -n "$cell $v: "; BP_LIB=$PWD/libs_ab/libbp_$v.so python bench.py --workload jitmv $cell --steps 60 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['call_us']['median'],1), 'frac', round(d['roofline']['frac'],3))"
done; done
