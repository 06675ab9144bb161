# ncu --set full of the config-2 kernels at the p = 0.05, 10 % cell (final state)
set -e
C="python bench.py --workload csrmv --law homo --p 0.05 --density 0.1 --steps 3 --warmup 3"
J="python bench.py --workload jitmv --law homo --p 0.05 --density 0.1 --steps 3 --warmup 3"
$C > /dev/null 2>&1 && $J > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_csr_stream -s 3 -c 1 -o gpurun_out/prof_csr_final $C > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:k_jit_tiled -s 3 -c 1 -o gpurun_out/prof_jit_final $J > /dev/null 2>&1
echo done
