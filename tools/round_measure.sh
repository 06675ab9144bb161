# all measurement cells of this round (run on the GPU box)
rm -f gpurun_out/net_all.jsonl gpurun_out/micro_all.jsonl
EXTRA=--no-cpu bash tools/net_cells.sh
for law in homo uniform; do for p in 0.001 0.01 0.05; do for d in 0.001 0.01 0.1; do
  python bench.py --workload csrmv --law $law --p $p --density $d --steps 100 --warmup 10 > gpurun_out/m.log 2>&1 && tail -1 gpurun_out/m.log >> gpurun_out/micro_all.jsonl
done; done; done
for law in homo uniform normal; do for p in 0.001 0.01 0.05; do for d in 0.001 0.01 0.1; do
  python bench.py --workload jitmv --law $law --p $p --density $d --steps 100 --warmup 10 > gpurun_out/m.log 2>&1 && tail -1 gpurun_out/m.log >> gpurun_out/micro_all.jsonl
done; done; done
echo measured
