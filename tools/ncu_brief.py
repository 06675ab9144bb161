"""Brief per-kernel summary of an .ncu-rep: duration, DRAM, issue, occupancy, top stalls."""
import csv, io, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
for v in rows[2:]:
    d = dict(zip(h, v))
    def f(k):
        try:
            return float(d.get(k, "nan").replace(",", ""))
        except ValueError:
            return float("nan")
    name = d.get("Kernel Name", "?")[:60]
    dur = f("gpu__time_duration.sum")
    rd, wr = f("dram__bytes_read.sum"), f("dram__bytes_write.sum")
    print(f"{name:60s} {dur:8.2f} us  dram r {rd:9.3f} w {wr:8.3f} MB  "
          f"issue {f('sm__inst_issued.avg.pct_of_peak_sustained_active'):5.1f}%  "
          f"occ {f('sm__warps_active.avg.pct_of_peak_sustained_active'):5.1f}%")
    st = {k.split("issue_stalled_")[1].split("_per")[0]: f(k) for k in d
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")}
    top = sorted(st.items(), key=lambda x: -x[1])[:5]
    print("    stalls:", ", ".join(f"{k} {v:.2f}" for k, v in top))
