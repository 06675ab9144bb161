# k_bin phases: the remote rows of an 8-GPU weak-scaling rank (188 k rows of
# the 100 M network, events restricted to the local 12.5 M segment), 4 lanes / warp
for S in 4 32 64; do echo "== remote S=$S"; LOCAL=1 tools/probes/probe_bin_new.bin 100000000 12500000 188000 $S | tail -3 | head -2; done
echo "== local cfg5 S=32"; tools/probes/probe_bin_new.bin 12500000 12500000 27500 32 | tail -3 | head -2
