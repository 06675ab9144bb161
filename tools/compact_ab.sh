# A/B: single-block compaction (default) vs memset + multi-block (BP_COMPACT_MULTI=1)
for cell in "csrmv --law homo --p 0.05" "csrmv --law uniform --p 0.05" "csrmv --law uniform --p 0.01" "csrmv --law homo --p 0.01" "jitmv --law homo --p 0.05" "jitmv --law homo --p 0.01"; do
 for v in "" 1; do
  echo -n "$cell multi=$v: "; BP_COMPACT_MULTI=$v python bench.py --workload $cell --density 0.1 --steps 60 | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['call_us']['median'],1), 'frac', round(d['roofline']['frac'],3))"
 done; done
