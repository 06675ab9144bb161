for r in 1 2; do
for v in t1024 t512 t768; do echo "== $v"; tools/probes/probe_bin_$v.bin 12500000 12500000 27500 32 | tail -3; done
echo "== t512x2"; GRID=296 tools/probes/probe_bin_t512x2.bin 12500000 12500000 27500 32 | tail -3
done
