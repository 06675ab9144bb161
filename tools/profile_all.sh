#!/bin/bash
# ncu evidence for profiles/ (run on the GPU box; each command first runs
# without ncu): default network workload launch list + full capture of the
# step kernels; CSR stream and JIT tiled microbench kernels.
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 300 --warmup 200 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 60 --csv \
    --log-file gpurun_out/launches_default.csv $CMD > /dev/null 2>&1
ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_step|k_bin_sorted" -s 600 -c 2 -o gpurun_out/prof_default -f $CMD > /dev/null 2>&1
CSR="python bench.py --workload csrmv --law homo --p 0.05 --density 0.1 --steps 10 --warmup 5"
$CSR > gpurun_out/prof_csr_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_csr_stream" -s 5 -c 1 \
    -o gpurun_out/prof_csr -f $CSR > /dev/null 2>&1
JIT="python bench.py --workload jitmv --law homo --p 0.05 --density 0.1 --steps 10 --warmup 5"
$JIT > gpurun_out/prof_jit_plain.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"k_jit_tiled" -s 5 -c 1 \
    -o gpurun_out/prof_jit -f $JIT > /dev/null 2>&1
echo done
