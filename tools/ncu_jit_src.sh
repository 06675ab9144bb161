# ncu --set full (source level) of k_jit_tiled, homogeneous weights, p = 0.05, 10 %
mkdir -p gpurun_out/jitsrc
ncu --set full --import-source on --clock-control none -k regex:k_jit_tiled -s 6 -c 1 -o gpurun_out/jitsrc/jit_homo -f \
  python bench.py --workload jitmv --law homo --p 0.05 --density 0.1 --steps 8 --warmup 3 --no-cpu --no-e2e > gpurun_out/jitsrc/log 2>&1
