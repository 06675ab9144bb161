# ncu evidence for the bench's default workload (run on the GPU box).
# 1) launch list of a short bench run, 2) full capture of the step kernels.
set -e
CMD="python bench.py --steps 300 --warmup 200 --no-cpu --no-e2e"
$CMD > gpurun_out/prof_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -s 600 -c 60 --csv \
    --log-file gpurun_out/launches_r01.csv $CMD > /dev/null 2>&1
ncu --set full --cache-control none --clock-control none --import-source on \
    -k regex:"k_step|k_bin_sorted" -s 600 -c 2 -o gpurun_out/prof_r01_f32 $CMD > /dev/null 2>&1
echo done
