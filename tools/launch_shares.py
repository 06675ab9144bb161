"""Per-kernel share of the timed steps from an ncu launch list
(`ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file F`):
sums gpu__time_duration per kernel name (cold-cache, serialised per launch --
the SHARES are what compares with the bench, not the absolute times).

    python tools/launch_shares.py launches.csv [out.json]
"""
import collections
import csv
import json
import sys


def shares(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    tot = collections.defaultdict(float)
    n = collections.Counter()
    for r in rows:
        if "Kernel Name" in r and "Metric Value" in r:
            hdr = r
            continue
        if hdr is None or len(r) < len(hdr):
            continue
        rec = dict(zip(hdr, r))
        if rec.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = rec["Kernel Name"].split("(")[0].replace("void ", "")
        unit = rec.get("Metric Unit", "nsecond")
        v = float(rec["Metric Value"].replace(",", ""))
        v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
        tot[name] += v
        n[name] += 1
    all_us = sum(tot.values())
    return {k: {"launches": n[k], "total_us": tot[k], "avg_us": tot[k] / n[k],
                "share": tot[k] / all_us} for k in sorted(tot, key=lambda k: -tot[k])}


if __name__ == "__main__":
    res = shares(sys.argv[1])
    print(json.dumps(res, indent=1))
    if len(sys.argv) > 2:
        json.dump(res, open(sys.argv[2], "w"), indent=1)
