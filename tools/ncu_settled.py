"""ncu --set full of the network step kernels in the SETTLED regime (run on
the GPU box): profiles the k_step and k_bin_sorted launches of the first
timed step of `bench.py --workload W --g G` (after its settle + warm-up
steps) and writes profiles/r02/ncu_settled_<W>_<G>.json with per-kernel
DRAM bytes, duration, issue utilisation and instruction counts -- the
`traffic` figure bench.py reports beside its roofline.

    python tools/ncu_settled.py [--workload coba_lif_jit] [--g f32]
"""
import argparse
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

METRICS = {
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__time_duration.sum": "duration",
    "smsp__inst_executed.sum": "inst_executed",
    "sm__inst_executed.avg.per_cycle_active": "ipc_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "lts__t_sectors_op_atom.sum": "l2_atom_sectors",
    "lts__t_sectors_op_red.sum": "l2_red_sectors",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9,
         "usecond": 1e-6, "msecond": 1e-3, "second": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="coba_lif_jit")
    ap.add_argument("--g", default="f32")
    ap.add_argument("--settle", type=int, default=None)
    ap.add_argument("--warmup", type=int, default=3)
    args = ap.parse_args()
    import bench
    settle = bench.settle_default(args.workload) if args.settle is None else args.settle
    os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
    rep = os.path.join(ROOT, "gpurun_out", f"ncu_settled_{args.workload}_{args.g}")
    skip = 2 * (settle + args.warmup)
    cmd = ["ncu", "--set", "full", "--clock-control", "none", "--import-source", "on",
           "-k", "regex:k_step|k_bin_sorted", "-s", str(skip), "-c", "2", "-f", "-o", rep,
           sys.executable, os.path.join(ROOT, "bench.py"), "--workload", args.workload,
           "--g", args.g, "--steps", "2", "--warmup", str(args.warmup), "--settle",
           str(settle), "--no-cpu", "--no-e2e"]
    subprocess.check_call(cmd, cwd=ROOT, stdout=subprocess.DEVNULL)
    raw = subprocess.check_output(["ncu", "-i", rep + ".ncu-rep", "--page", "raw", "--csv"],
                                  text=True)
    rows = list(csv.reader(io.StringIO(raw)))
    head, units, data = rows[0], rows[1], rows[2:]
    out = {"workload": args.workload, "g": args.g, "settle_steps": settle,
           "command": " ".join(cmd[:-12]) + " ... bench.py --workload %s --g %s" % (
               args.workload, args.g),
           "kernels": {}}
    for r in data:
        name = r[head.index("Kernel Name")]
        key = "k_step" if "k_step" in name else (
            "k_bin_sorted" if "k_bin_sorted" in name else name)
        rec = {"name": name}
        for m, short in METRICS.items():
            if m in head:
                i = head.index(m)
                try:
                    v = float(r[i].replace(",", ""))
                except ValueError:
                    continue
                if short == "duration":
                    rec["duration_unit"] = units[i]
                    rec[short] = v
                else:
                    rec[short] = v * SCALE.get(units[i], 1.0)
        if "dram_read" in rec and "dram_write" in rec:
            rec["dram_bytes"] = rec["dram_read"] + rec["dram_write"]
        out["kernels"][key] = rec
    dst = os.path.join(ROOT, "profiles", "r02", f"ncu_settled_{args.workload}_{args.g}.json")
    with open(dst, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
