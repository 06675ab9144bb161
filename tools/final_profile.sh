# Round-end evidence for profiles/r02: default bench lines, the ncu launch
# list of the timed region of the same command (kernel shares), and one
# ncu --set full capture of the settled step kernels (bench.py's `traffic`).
O=gpurun_out/final
mkdir -p $O
python bench.py --steps 20 --warmup 5 > $O/bench_20.json 2> $O/bench_20.err
python bench.py --steps 2000 --warmup 5 --no-cpu > $O/bench_2000.json 2> $O/bench_2000.err
# launch list: skip the 2 x (settle 2000 + warm-up 5) launches, then 2 x 100 steps
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_step|k_bin" -s 4010 -c 200 \
    --csv --log-file $O/launches.csv python bench.py --steps 100 --warmup 5 --no-cpu --no-e2e \
    > $O/ncu_launches.log 2>&1
python tools/launch_shares.py $O/launches.csv $O/launch_shares.json > /dev/null
python tools/ncu_settled.py --workload coba_lif_jit --g f32 > $O/ncu_settled.log 2>&1
cp profiles/r02/ncu_settled_coba_lif_jit_f32.json $O/ 2>/dev/null
for wl in coba4m_jit hh400k_csr coba4000_csr coba4m_k1000 coba4m_p001; do
  python bench.py --workload $wl --steps 400 --warmup 5 --no-cpu --no-e2e > $O/bench_$wl.json 2>&1
done
for g in fix32 fix64; do
  python bench.py --g $g --steps 400 --warmup 5 --no-cpu --no-e2e > $O/bench_$g.json 2>&1
done
python bench.py --emulate-world 8 --steps 400 --warmup 20 > $O/emulate_g8.json 2>&1
python bench.py --emulate-world 2 --steps 400 --warmup 20 > $O/emulate_g2.json 2>&1
python bench.py --impl reference --steps 5 --warmup 3 > $O/reference.json 2>&1
echo done > $O/done
