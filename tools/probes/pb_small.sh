for S in 2 4 8; do echo "== remote S=$S"; LOCAL=1 tools/probes/probe_bin_new.bin 100000000 12500000 188000 $S | tail -2 | head -1; done
for S in 2 4 8; do echo "== local G8 S=$S"; LOCAL=1 tools/probes/probe_bin_new.bin 100000000 12500000 27000 $S | tail -2 | head -1; done
