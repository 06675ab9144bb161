for r in 1 2; do for v in old new; do
 echo "== $v"; tools/probes/probe_bin_$v.bin 12500000 12500000 27500 32 | tail -3
 tools/probes/probe_bin_$v.bin 4000000 500000 8800 4 | tail -3
done; done
