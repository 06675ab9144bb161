# k_csr_stream phase timing (globaltimer marks) on the three judged config-2 cells
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o /tmp/probe_csr tools/probes/probe_csr.cu || exit 1
/tmp/probe_csr 0.05 0.1 1 1 | tail -3
/tmp/probe_csr 0.05 0.1 0 1 | tail -3
/tmp/probe_csr 0.01 0.1 0 1 | tail -3
/tmp/probe_csr 0.01 0.1 1 1 | tail -3
