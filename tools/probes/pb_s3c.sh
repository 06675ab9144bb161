# k_bin phases for Fig S3C (4 M, p = 0.001 -> K = 1999, 410 rows, seg n/8) and S3B (K = 7999)
for S in 4 32 64; do
  echo "== S3C S=$S"; tools/probes/probe_bin_new.bin 4000000 500000 410 $S 1999 | tail -2 | head -1
  echo "== S3B S=$S"; tools/probes/probe_bin_new.bin 4000000 500000 1640 $S 7999 | tail -2 | head -1
done
