# A/B: bench f32 default with alternative library builds: bash tools/ab.sh libA.so libB.so ...
for lib in "$@"; do
  BP_LIB=$PWD/paper_2311_05106_b200/$lib python bench.py --g ${G:-f32} --steps 2000 --warmup 200 --no-cpu --no-e2e > gpurun_out/ab.log 2>&1
  python - "$lib" <<'PY'
import json, sys
d = json.loads(open("gpurun_out/ab.log").read().strip().splitlines()[-1]); r = d["roofline"]
print(sys.argv[1], "us/step=%.1f" % (d["ms_per_step"] * 1e3), "kern=%.1f" % r["avg_launch_us"], "bin=%.1f" % r["bin_kernel_avg_us"])
PY
done
