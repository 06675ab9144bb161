# Pipe-level utilisation of the issue/ALU-bound kernels (k_jit_tiled per law,
# k_bin_sorted at config 5, k_csr_stream): which execution pipe binds.
#   bash tools/ncu_pipes.sh OUTDIR
O=${1:-gpurun_out/pipes}; mkdir -p $O
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,\
sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_uniform.avg.pct_of_peak_sustained_active,\
sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
for law in homo uniform normal; do
  ncu --metrics $M --clock-control none -k regex:k_jit -s 6 -c 1 --csv --log-file $O/jit_$law.csv \
    python bench.py --workload jitmv --law $law --p 0.05 --density 0.1 --steps 8 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
done
ncu --metrics $M --clock-control none -k regex:k_csr_stream -s 6 -c 1 --csv --log-file $O/csr_hetero.csv \
  python bench.py --workload csrmv --p 0.05 --density 0.1 --steps 8 --warmup 3 --no-cpu --no-e2e > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_bin_sorted -s 2 -c 1 --csv --log-file $O/bin_cfg5.csv \
  tools/probes/probe_bin_new.bin 12500000 12500000 27500 32 > /dev/null 2>&1
ncu --metrics $M --clock-control none -k regex:k_step_persist -s 2010 -c 1 --csv --log-file $O/kstep_cfg5.csv \
  python bench.py --steps 20 --warmup 3 --settle 2000 --no-cpu --no-e2e > /dev/null 2>&1
ls -la $O
