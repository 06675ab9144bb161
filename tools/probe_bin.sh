# k_bin_sorted phase timing (globaltimer marks) for the network shapes
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/probe_bin tools/probes/probe_bin.cu || exit 1
for S in 4 8 32; do
  /tmp/probe_bin 12500000 12500000 27500 $S | tail -2      # config 5, G = 1
  /tmp/probe_bin 4000000 500000 8800 $S | tail -2          # config 3, seg n/8
done
