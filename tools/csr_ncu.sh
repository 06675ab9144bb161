#!/bin/bash
# ncu --set full of k_csr_tiled on the p=0.05, d=10% microbench cells (homo, uniform)
set -e
python -c "import __graft_entry__ as g; g.build_lib()"
mkdir -p gpurun_out
for law in homo uniform; do
  python bench.py --workload csrmv --law $law --p 0.05 --density 0.1 --steps 20 --warmup 5 > gpurun_out/csr_$law.log 2>&1
  tail -1 gpurun_out/csr_$law.log | cut -c1-300
  ncu --set full --clock-control none --import-source on -k regex:"k_csr_(tiled|stream|split|reduce)" -s 12 -c 4 \
      -o gpurun_out/csr_$law -f python bench.py --workload csrmv --law $law --p 0.05 --density 0.1 --steps 3 --warmup 3 > gpurun_out/csr_ncu_$law.log 2>&1 || tail -5 gpurun_out/csr_ncu_$law.log
done
