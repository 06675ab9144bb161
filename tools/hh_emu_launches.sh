# ncu launch list of the emulated HH 400k strong-scaling rank step (G = 1 / 2)
mkdir -p gpurun_out/hhemu
for G in 1 2; do
  if [ $G = 1 ]; then A=""; else A="--emulate-world $G --no-graph"; fi
  ncu --metrics gpu__time_duration.sum --clock-control none -s 100 -c 60 --csv \
      --log-file gpurun_out/hhemu/g$G.csv python bench.py --workload hh400k_csr $A --steps 40 --warmup 30 --no-cpu --no-e2e > gpurun_out/hhemu/g$G.log 2>&1
  python tools/launch_shares.py gpurun_out/hhemu/g$G.csv gpurun_out/hhemu/g$G.json
done
