# ncu --set full of k_bin_sorted in the settled regime for each BP_BIN_GROUP
# given (default 4 32), reports to gpurun_out/ncu_bin_S<g>.ncu-rep
WL=${WL:-coba_lif_jit}
for g in ${GROUPS:-4 32}; do
  BP_BIN_GROUP=$g ncu --set full --clock-control none --import-source on -k regex:k_bin_sorted \
    -s 2005 -c 1 -f -o gpurun_out/ncu_bin_${WL}_S$g python bench.py --workload $WL --steps 2 \
    --warmup 3 --settle 2000 --no-cpu --no-e2e > /dev/null 2>&1
  echo "S=$g rc=$?"
done
