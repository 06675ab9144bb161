# ncu evidence for the gap samplers (NEXT 4): instructions per regenerated
# gap of k_jit_rows (uniform vs geometric) and a full capture of the
# geometric k_jit_tiled on the p = 0.05, 10 % cell.
set -e
A="--workload jitrows --p 0.05 --steps 3 --warmup 3"
B="--workload jitmv --law homo --gap geometric --p 0.05 --density 0.1 --steps 3 --warmup 3"
python bench.py $A --gap uniform > gpurun_out/geo_plain_u.log 2>&1 && \
python bench.py $A --gap geometric > gpurun_out/geo_plain_g.log 2>&1 && \
python bench.py $B > gpurun_out/geo_plain_t.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_jit_rows -c 2 --csv --log-file gpurun_out/ncu_rows_u.csv python bench.py $A --gap uniform > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_alu.sum,sm__inst_executed_pipe_fma.sum,sm__inst_executed_pipe_fmaheavy.sum,smsp__issue_active.avg.pct_of_peak_sustained_active --clock-control none -k regex:k_jit_rows -c 2 --csv --log-file gpurun_out/ncu_rows_g.csv python bench.py $A --gap geometric > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_jit_tiled -s 3 -c 1 -o gpurun_out/prof_jit_tiled_geo python bench.py $B > /dev/null 2>&1
echo done
