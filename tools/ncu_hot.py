"""Hottest SASS instructions (warp-stall samples) of one kernel in an .ncu-rep."""
import csv, io, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
n = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass",
                      "-k", f"regex:{kern}"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Address"][0]
h = rows[hi]
ci = h.index("Warp Stall Sampling (All Samples)")
ex = h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) > ci and r[0].startswith("0x") is False and not r[0][:1].isdigit():
        continue
    try:
        data.append((float(r[ci] or 0), int(float(r[ex] or 0)), r[0], r[1][:80]))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data) or 1
for d in sorted(data, reverse=True)[:n]:
    print("%5.1f%% %10d %s %s" % (100 * d[0] / tot, d[1], d[2], d[3]))
