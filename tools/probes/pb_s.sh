for r in 1 2; do for S in 32 16 8 4; do
 echo "== cfg5 S=$S"; tools/probes/probe_bin_s.bin 12500000 12500000 27500 $S | tail -3
done
for S in 32 16 8 4; do echo "== cfg3 seg n/8 S=$S"; tools/probes/probe_bin_s.bin 4000000 500000 8800 $S | tail -3; done
for S in 32 16 8 4; do echo "== cfg3 seg n S=$S"; tools/probes/probe_bin_s.bin 4000000 4000000 8800 $S | tail -3; done
done
