# local binning grid of a partitioned rank (few events per block): 148 vs fewer blocks
run() { python bench.py --steps 400 --warmup 5 --no-cpu --no-e2e "$@" | python -c "
import json,sys; d=json.loads([l for l in sys.stdin if l.startswith('{')][-1]); print(round(d['ms_per_step']*1e3,2))"; }
for G in 8 2; do for r in 1 2; do for g in 148 74 37; do
  echo -n "G=$G local grid $g: "; BP_BIN_GRID_LOCAL=$g run --emulate-world $G
done; done; done
for g in 148 74; do echo -n "G=1 local grid $g: "; BP_BIN_GRID_LOCAL=$g run; done
