# k_bin phases of the item paths: remote rows of an 8-GPU rank, config 3 (seg n/8), Fig S3C / S3B
echo "== remote S=4"; LOCAL=1 tools/probes/probe_bin_new.bin 100000000 12500000 188000 4 | tail -2 | head -1
echo "== cfg3 S=4"; tools/probes/probe_bin_new.bin 4000000 500000 8800 4 | tail -2 | head -1
echo "== S3C S=64"; tools/probes/probe_bin_new.bin 4000000 500000 410 64 1999 | tail -2 | head -1
echo "== S3B S=64"; tools/probes/probe_bin_new.bin 4000000 500000 1640 64 7999 | tail -2 | head -1
echo "== cfg5 S=32"; tools/probes/probe_bin_new.bin 12500000 12500000 27500 32 | tail -2 | head -1
