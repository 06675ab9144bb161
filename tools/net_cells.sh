for wl in ${WLS:-coba4000_csr coba4m_jit hh400k_csr coba_lif_jit}; do for m in "--g fix64" "--g fix32" "--g f32"; do
python bench.py --workload $wl --steps ${STEPS:-2000} --warmup 200 --no-e2e $m $EXTRA > gpurun_out/n.log 2>&1 || { tail -5 gpurun_out/n.log; continue; }
cat gpurun_out/n.log | tail -1 >> gpurun_out/net_all.jsonl
python - "$wl" "$m" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/n.log").read().strip().splitlines()[-1]); r = d["roofline"]
c = d.get("cpu_baseline") or {}
print(sys.argv[1], sys.argv[2][4:], "us/step=%.2f" % (d["ms_per_step"] * 1e3), "Gev/s=%.2f" % (d["value"] / 1e9),
      "sim=%.2f" % d["sim_s_per_wall_s"], "kern_us=%.1f" % r["avg_launch_us"], "frac=%.3f" % r["frac"],
      "ev/step=%d" % d["events_per_step"], "cpu_Mev/s=%.2f" % (c.get("value", 0) / 1e6))
PY
done; done
