# quick bench summary lines: fixed and fp32 modes
for m in "--g fix64" "--g fix32" "--g f32"; do
  python bench.py --steps ${STEPS:-2000} --warmup 200 --no-cpu --no-e2e $m $EXTRA > gpurun_out/b${m#--g }.log 2>&1
  python - "$m" <<'PY'
import json, sys
m = sys.argv[1]
d = json.loads(open(f"gpurun_out/b{m[4:]}.log").read().strip().splitlines()[-1])
r = d["roofline"]
print(m[4:], "us/step=%.1f" % (d["ms_per_step"] * 1e3), "Gev/s=%.2f" % (d["value"] / 1e9),
      "step_kernel_us=%.1f" % r["avg_launch_us"], "share=%.2f" % r["share_of_step"], "bin_us=%.1f" % r["bin_kernel_avg_us"],
      "frac=%.3f" % r["frac"], "ev/step=%d" % d["events_per_step"], "sim=%.3f" % d["sim_s_per_wall_s"])
PY
done
