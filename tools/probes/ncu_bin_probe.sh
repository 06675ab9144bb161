# one ncu --set full capture of k_bin_sorted in the phase probe (config 5, warp-per-row)
mkdir -p gpurun_out/$1
ncu --set full --import-source on --clock-control none -k k_bin_sorted -s 2 -c 1 -o gpurun_out/$1/kbin_probe -f \
  tools/probes/probe_bin_new.bin 12500000 12500000 27500 32
