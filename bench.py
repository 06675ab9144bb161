"""bench.py -- synaptic events/s and simulated-s per wall-s of the COBA E/I
network on 1/2/4/8 B200 (BASELINE.json metric, config 5 shape).

Workload (default, `--workload coba_lif_jit`): Listing S3's COBA-LIF E/I
network with JIT connectivity (event_mv_prob_homo), fan-in
80 (p = 80/N), 12.5 M neurons per GPU (weak scaling: N = 12.5M x G),
dt = 0.1 ms, fixed-point int64 conductances (rule F1).  One "step" = one
0.1 ms timestep of the whole hot path: spike delivery (JIT regeneration +
scatter), fused Expon + COBA + LIF update, spike compaction, and for G > 1
the bit-packed spike all-gather.  State per GPU is 525 MB > 126 MB L2, so
no L2 flush is needed between steps (inputs larger than L2).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import math
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DT_MS = 0.1
N_PER_GPU = 12_500_000
METRIC = "synaptic events/sec & sim-sec per wall-sec, COBA E/I at 1/2/4/8 B200"
UNIT = "synaptic events/s"
# algorithmic bytes of the fused step kernel (k_step): per neuron V r+w (8),
# refractory counter r (1), g_E + g_I r+w (32 fixed point / 16 fp32); per
# synaptic event one 4-byte bucket record written and read back (8); per
# neuron 1/8 byte of spike bits.
def step_bytes(n_local, events_per_step, fixed):
    """k_step: state r+w + the 4-byte bucket record of every incoming event."""
    per_neuron = 8 + 1 + (32 if fixed else 16) + 0.125
    return per_neuron * n_local + 4 * events_per_step


def _ncu_traffic(kernel_prefix):
    """dram__bytes_read + dram__bytes_write per launch of `kernel_prefix` from
    the committed ncu --set full capture of this round (profiles/r01), or None."""
    path = os.path.join(ROOT, "profiles", "r01", "ncu_full_f32_default.json")
    try:
        with open(path) as f:
            rows = json.load(f)
    except (OSError, ValueError):
        return None
    for r in rows:
        if r.get("Kernel Name", "").startswith(kernel_prefix):
            rd = float(r["dram__bytes_read.sum"].split()[0])
            wr = float(r["dram__bytes_write.sum"].split()[0])
            unit = r["dram__bytes_read.sum"].split()[1] if " " in r["dram__bytes_read.sum"] else "byte"
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)
            return (rd + wr) * scale
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


class ClockSampler:
    """SM clocks + throttle reasons sampled in-process through NVML (a
    background thread, every 5 ms) from before the warm-up to after the
    timed region, so even a millisecond-long timed region has samples on
    both sides of it; mark() brackets the timed region (host clock) and the
    summary reports the samples inside it and around it.  Falls back to a
    `nvidia-smi -lms 100` subprocess when NVML is unavailable."""
    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20,
               "hw_thermal_slowdown": 0x40, "sw_power_cap": 0x4,
               "hw_power_brake_slowdown": 0x80}

    def __init__(self, index: int, period_s: float = 0.005):
        self.index, self.period = index, period_s
        self.samples = []               # (t, sm_mhz, reasons bitmask)
        self.max_mhz = None
        self.t0 = self.t1 = None
        self._stop = None
        self._thread = None
        self.source = None

    def _handle(self):
        import pynvml
        pynvml.nvmlInit()
        try:
            import torch
            pr = torch.cuda.get_device_properties(self.index)
            bus = "%08x:%02x:%02x.0" % (pr.pci_domain_id, pr.pci_bus_id, pr.pci_device_id)
            return pynvml, pynvml.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            return pynvml, pynvml.nvmlDeviceGetHandleByIndex(self.index)

    def __enter__(self):
        import threading
        try:
            nv, h = self._handle()
            self.max_mhz = float(nv.nvmlDeviceGetMaxClockInfo(h, nv.NVML_CLOCK_SM))
            self.source = "nvml"
        except Exception:
            nv = h = None
            self.source = "none"
        self._stop = threading.Event()

        def run():
            while not self._stop.is_set():
                try:
                    sm = float(nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM))
                    rs = int(nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                    self.samples.append((time.perf_counter(), sm, rs))
                except Exception:
                    return
                self._stop.wait(self.period)
        if h is not None:
            self._thread = threading.Thread(target=run, daemon=True)
            self._thread.start()
        return self

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_stop(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        if self._thread is not None:
            self._stop.set()
            self._thread.join(timeout=2)
        return False

    def summary(self):
        t0 = self.t0 if self.t0 is not None else -1e30
        t1 = self.t1 if self.t1 is not None else 1e30
        inside = [s for s in self.samples if t0 <= s[0] <= t1]
        # a short timed region: the samples of the 50 ms on each side of it
        near = inside or [s for s in self.samples if t0 - 0.05 <= s[0] <= t1 + 0.05]
        reasons = set()
        for _, _, rs in near:
            for nm, bit in self.REASONS.items():
                if rs & bit:
                    reasons.add(nm)
        sm = [x[1] for x in near]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": self.max_mhz,
                "reasons": sorted(reasons), "samples": len(near),
                "samples_in_timed_region": len(inside), "samples_total": len(self.samples),
                "source": self.source,
                "window": ("inside the timed region" if inside else
                           "within 50 ms of the timed region (region shorter than the period)")}


# ---------------------------------------------------------------------------
# CPU oracle leg (cpu_baseline and --impl reference): the oracle as it stands
# ---------------------------------------------------------------------------

def oracle_sample_steps(n_total: int, n_steps: int, fraction: float, seed: int = 7,
                        wl: str = "coba_lif_jit", count_events: bool = True):
    """Time the oracle on a bounded sample of the same workload: each step
    delivers the spikes of `fraction` of the presynaptic rows (all of their
    events, E and I projections, Bernoulli(22 Hz * dt) activity -- the
    oracle network's measured rate) and updates `fraction` of the neurons.
    Returns (seconds, events, neuron_updates)."""
    import numpy as np

    import oracle
    from paper_2311_05106_b200 import inputs
    from paper_2311_05106_b200.network import SEED_E, SEED_I
    oracle.build()
    n_exc = n_total * 4 // 5
    p, w_e, w_i = net_params(wl, n_total)
    K = oracle.conn_len(p)
    je = oracle.JitSpec(SEED_E, K, n_total, oracle.LAW_HOMO, w_e)
    ji = oracle.JitSpec(SEED_I, K, n_total, oracle.LAW_HOMO, w_i)
    n_rows_e = max(1, int(n_exc * fraction))
    n_rows_i = max(1, int((n_total - n_exc) * fraction))
    n_upd = max(32, int(n_total * fraction))
    v = inputs.lif_v0(n_upd)
    ref = np.zeros(n_upd, np.uint8)
    g_e = np.zeros(n_total, np.int64)
    g_i = np.zeros(n_total, np.int64)
    params = oracle.lif_params()
    density = 22.0 * DT_MS * 1e-3
    patterns = [(inputs.spike_pattern(n_rows_e, density, seed + 2 * k),
                 inputs.spike_pattern(n_rows_i, density, seed + 2 * k + 1))
                for k in range(min(n_steps, 8))]
    t0 = time.perf_counter()
    for k in range(n_steps):
        ev_e, ev_i = patterns[k % len(patterns)]
        oracle.jit_event_mv(je, n_rows_e, n_total, ev_e, out_kind=oracle.OUT_FIX, out=g_e)
        oracle.jit_event_mv(ji, n_rows_i, n_total, ev_i, out_kind=oracle.OUT_FIX, out=g_i)
        oracle.lif_step(params, v, g_e[:n_upd], g_i[:n_upd], ref)
    secs = time.perf_counter() - t0
    if not count_events:
        return secs, None, n_upd * n_steps
    # events delivered (outside the timed region): fan-out of every active row
    per_pattern = []
    for ev_e, ev_i in patterns:
        e = 0
        for spec, ev in ((je, ev_e), (ji, ev_i)):
            for r in np.nonzero(ev)[0]:
                e += len(oracle.jit_row(spec, n_total, int(r))[0])
        per_pattern.append(e)
    events = sum(per_pattern[k % len(patterns)] for k in range(n_steps))
    return secs, events, n_upd * n_steps


def oracle_full_network(wl, n_total, csr, n_steps):
    """The oracle's own run_network (rule S1) on the workload's network for
    n_steps; returns (seconds, events)."""
    import numpy as np

    import oracle
    from paper_2311_05106_b200 import inputs
    from paper_2311_05106_b200.network import SEED_E, SEED_I
    spec = NETWORKS[wl]
    n = n_total
    n_exc = n * 4 // 5
    p, w_e, w_i = net_params(wl, n)
    K = oracle.conn_len(p)
    w = (w_e, w_i)
    if csr is None:
        pe = oracle.Projection(0, n_exc, jit=oracle.JitSpec(SEED_E, K, n, oracle.LAW_HOMO, w[0]))
        pi = oracle.Projection(n_exc, n - n_exc, jit=oracle.JitSpec(SEED_I, K, n, oracle.LAW_HOMO, w[1]))
        fan = [np.array([len(oracle.jit_row(p.jit, n, r)[0]) for r in range(p.n_rows)])
               for p in (pe, pi)] if n <= 200_000 else None
    else:
        (ipe, ixe), (ipi, ixi) = [(a.cpu().numpy(), b.cpu().numpy()) for a, b in csr]
        pe = oracle.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=w[0])
        pi = oracle.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=w[1])
        fan = [np.diff(ipe), np.diff(ipi)]
    if spec["model"] == "lif":
        st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
                  ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
        params = oracle.lif_params()
    else:
        v, m, h, nk = inputs.hh_init(n)
        st = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
                  spikes=np.zeros(n, np.uint8))
        params = oracle.hh_params()
    t0 = time.perf_counter()
    raster = oracle.run_network(spec["model"], params, st, pe, pi, n_steps)
    secs = time.perf_counter() - t0
    # events: spikes of step k are delivered at step k+1
    fan_all = np.concatenate(fan)
    events = int((raster[:-1].astype(np.int64) @ fan_all).sum()) if fan is not None else 0
    return secs, events


def _cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_baseline(wl, n_total, csr, budget_s: float = 15.0):
    if n_total > 1_000_000:
        fraction = 1.0 / 32
        secs, events, _ = oracle_sample_steps(n_total, 2, fraction, wl=wl)   # calibrate
        per_step = max(secs / 2, 1e-3)
        steps = max(2, min(5000, int(budget_s / per_step)))
        secs, events, upd = oracle_sample_steps(n_total, steps, fraction, wl=wl)
        out = {"value": events / secs, "unit": UNIT, "cores": 1, "kind": "oracle",
               "sample": (f"{steps} steps of the {n_total:,}-neuron network with 1/32 of "
                          f"presynaptic rows active-eligible (Bernoulli 22 Hz x dt) and 1/32 "
                          f"of neurons updated per step; {events:,} events in {secs:.1f} s, "
                          f"single-threaded C oracle"),
               "sim_s_per_wall_s_equiv": (steps * DT_MS * 1e-3 * fraction) / secs,
               "cpu_model": _cpu_model()}
        # the same sample with the oracle's host threads on every core (its
        # order-free loops; bit-identical results -- SURVEY 8(d) asks for
        # both timings)
        import oracle
        cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
        if cores and cores > 1:
            oracle.set_threads(cores)
            try:
                secs_t, _, _ = oracle_sample_steps(n_total, steps, fraction, wl=wl,
                                                   count_events=False)
            finally:
                oracle.set_threads(1)
            out["all_cores"] = {"value": events / secs_t, "unit": UNIT, "cores": cores,
                                "kind": "oracle (host threads)",
                                "sample": f"the same {steps} steps; {events:,} events in "
                                          f"{secs_t:.1f} s"}
        return out
    secs, _ = oracle_full_network(wl, n_total, csr, 20)                 # calibrate
    steps = max(21, min(10_000, int(budget_s / max(secs / 20, 1e-6))))
    secs, events = oracle_full_network(wl, n_total, csr, steps)
    return {"value": events / secs, "unit": UNIT, "cores": 1, "kind": "oracle",
            "sample": (f"the full {n_total:,}-neuron network for {steps} steps "
                       f"({steps * DT_MS:.0f} ms simulated) through the oracle's run_network "
                       f"(rule S1), single-threaded C oracle; {events:,} events in {secs:.1f} s"),
            "sim_s_per_wall_s": steps * DT_MS * 1e-3 / secs}


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    n_total = N_PER_GPU * args.gpus
    fraction = 1.0 / 64
    # the oracle with its host threads on every core of the box (its
    # order-free loops; bit-identical to one thread)
    import oracle
    oracle.build()
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    cores = max(1, cores or 1)
    oracle.set_threads(cores)
    _, _, _ = oracle_sample_steps(n_total, max(1, args.warmup), fraction, count_events=False)
    secs, events, upd = oracle_sample_steps(n_total, args.steps, fraction)
    oracle.set_threads(1)
    value = events / secs
    sample = (f"each step: 1/64 of the presynaptic rows (Bernoulli 22 Hz x dt) of the "
              f"{n_total:,}-neuron network delivered through the oracle's Listing S2 "
              f"loop + 1/64 of the neurons updated (rule N1); {cores} host threads "
              f"({_cpu_model()})")
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f32+i64fix",
            "data": "synthetic",
            "config": {"workload": "coba_lif_jit", "n_per_gpu": N_PER_GPU,
                       "n_total": n_total, "fan_in": 80, "dt_ms": DT_MS},
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
# Network workloads (BASELINE.json configs).  The default, config 5, is the
# one the metric is quoted on ("COBA E/I at 1/2/4/8 B200", weak scaling).
NETWORKS = {
    "coba_lif_jit": dict(model="lif", conn="jit", per_gpu=N_PER_GPU, scaling="weak",
                         cfg="config 5: COBA-LIF JIT, 12.5M neurons per GPU, postsynaptic partition"),
    "coba4m_jit": dict(model="lif", conn="jit", n=4_000_000, scaling="strong", seg8=True,
                       cfg="config 3: COBA-LIF JIT 4M neurons, fan-in 80"),
    "coba4000_csr": dict(model="lif", conn="csr", n=4000, scaling="strong",
                         cfg="config 1: COBA-LIF 4000 neurons (3200E/800I), p=0.02, CSR"),
    "hh400k_csr": dict(model="hh", conn="csr", n=400_000, scaling="strong",
                       cfg="config 4: COBA-HH 400k neurons, fan-in 80, CSR"),
    "coba100m_jit": dict(model="lif", conn="jit", n=100_000_000, scaling="strong", seg8=True,
                         cfg="config 5 total size on ONE GPU: COBA-LIF JIT 1e8 neurons, fan-in 80"),
    # Fig S3B / S3C regimes at the config-3 size
    "coba4m_k1000": dict(model="lif", conn="jit", n=4_000_000, scaling="strong", fan_in=1000,
                         seg8=True,
                         cfg="Fig S3B: COBA-LIF JIT 4M neurons, 1000 synapses per neuron, "
                             "weights x 80/1000"),
    "coba4m_p001": dict(model="lif", conn="jit", n=4_000_000, scaling="strong", p=0.001,
                        seg8=True,
                        cfg="Fig S3C: COBA-LIF JIT 4M neurons, fixed p = 0.001 (fan-in 4000), "
                            "weights x 80/4000"),
}


def net_params(wl, n):
    """(p, w_exc, w_inh) of a workload: fan-in 80 unless the workload
    sets `fan_in` (Fig S3B) or a fixed `p` (Fig S3C); then the weights are
    rescaled by 80 / fan-in (reading R29: the mean synaptic drive K w of
    P:974-981 is kept)."""
    spec = NETWORKS[wl]
    w = (0.6, 6.7) if spec["model"] == "lif" else (6.0, 67.0)
    if "p" in spec:
        p = spec["p"]
    else:
        p = spec.get("fan_in", 80) / n
    scale = 80.0 / (p * n) if ("p" in spec or "fan_in" in spec) else 1.0
    return p, w[0] * scale, w[1] * scale


def network_size(wl, world):
    spec = NETWORKS[wl]
    return spec["per_gpu"] * world if "per_gpu" in spec else spec["n"]


def seg_len_of(wl, n):
    """JIT segment length (rule J4).  Weak scaling (config 5): the 12.5 M
    neurons of one GPU, so each rank regenerates only its own segment.
    Strong-scaling JIT configs: n / 8 at EVERY GPU count (the 8-GPU
    partition), so G = 1, 2, 4, 8 simulate the same connectivity."""
    spec = NETWORKS[wl]
    if spec.get("seg8"):
        return -(-n // 8 // 32) * 32
    return spec.get("per_gpu", n) if "per_gpu" in spec else n


def build_network(wl, world, rank, fixed, dev, exchange="caller"):
    """The workload's network; CSR connectivity = materialise(JIT spec) with
    the library's own generator ('CSR = materialise(jit spec)')."""
    import paper_2311_05106_b200 as bp
    from paper_2311_05106_b200.network import SEED_E, SEED_I, CobaNetwork
    spec = NETWORKS[wl]
    n = network_size(wl, world)
    csr = None
    if spec["conn"] == "csr":
        n_exc = n * 4 // 5
        p = net_params(wl, n)[0]
        ipe, ixe, _ = bp.jitconn_materialize(bp.jitconn_spec(SEED_E, p), n_exc, n,
                                             with_data=False, device=dev)
        ipi, ixi, _ = bp.jitconn_materialize(bp.jitconn_spec(SEED_I, p), n - n_exc, n,
                                             with_data=False, device=dev)
        csr = ((ipe, ixe), (ipi, ixi))
    p, w_e, w_i = net_params(wl, n)
    seg = seg_len_of(wl, n) if spec["conn"] == "jit" else None
    return CobaNetwork(n, model=spec["model"], conn=spec["conn"], fixed=fixed, rank=rank,
                       world=world, device=dev, csr=csr, p=p, w_exc=w_e, w_inh=w_i,
                       seg_len=seg, exchange=exchange), csr


def state_bytes_per_neuron(model, fixed):
    g = 32 if fixed is True else 16
    return (8 + 1 if model == "lif" else 32) + g + 0.125


# Measured lane instructions per regenerated gap of the paper's U[1, K]
# sampler (ncu smsp__inst_executed x 32 / gaps of a k_jit_rows call:
# profiles/r01/ncu_gap_samplers.json) -- the algorithmic core of the network
# binning kernel (regeneration); staging, sort and the bucket writes are on
# top of it, so the k_bin "alu" fraction below is that core's share of the
# issue roof.
BIN_CORE_OPS_PER_EVENT = 27.4


def _ncu_traffic_r02(wl, g, kernel_prefix):
    """DRAM bytes (read + write) per launch of `kernel_prefix` from the
    committed ncu --set full capture of THIS workload in the settled regime
    (profiles/r02/ncu_settled_<wl>_<g>.json, written by
    tools/ncu_settled.py from an ncu run that skips the settle steps), or
    None when no such capture exists."""
    path = os.path.join(ROOT, "profiles", "r02", f"ncu_settled_{wl}_{g}.json")
    try:
        with open(path) as f:
            rec = json.load(f)
    except (OSError, ValueError):
        return None, None
    k = rec.get("kernels", {}).get(kernel_prefix)
    if not k:
        return None, None
    return float(k["dram_bytes"]), os.path.relpath(path, ROOT)


def launches_per_step(model: str, n_local: int, n_total: int, world: int,
                      sms: int = 148) -> int:
    """libbp kernel launches per network step (bp_api.cu launch_step and
    remote_scatter): the update kernel; the local binning unless the dense HH
    update delivers its own spikes (n_local <= 2^21); for world > 1 the
    remote binning -- one launch when each binning block's share of the
    remote spike words is <= 1024 words (bin_spike_range's listing rule),
    else compaction + binning."""
    dense_hh = model == "hh" and n_local <= (2 << 20)
    n = 1 if dense_hh else 2
    if world > 1:
        remote_words = (n_total - n_local + 31) // 32
        n += 1 if remote_words <= sms * 1024 else 2
    return n


def settle_default(wl):
    """Untimed pre-roll: the network starts from V0 ~ N(-55, 2),
    every neuron crosses threshold within the first ~30 steps and the
    synchronous burst and its echoes (up to ~15 M events per step at 12.5 M
    neurons, 7x the settled load) fade over the first few hundred steps; the
    timed region starts in the settled asynchronous regime."""
    return 0 if network_size(wl, 1) <= 4096 else 2000


def run_ours(args):
    import torch
    import torch.distributed as dist

    import __graft_entry__ as ge
    ge.build_lib()

    wl = args.workload
    spec = NETWORKS[wl]
    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # one GPU per rank; --dist-backend gloo lets several ranks share a GPU for
    # a functional check of the N > 1 path (host-mediated exchange)
    device_index = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(device_index)
    dev = torch.device("cuda", device_index)
    if world > 1:
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group("gloo")
    n_total = network_size(wl, world)
    fixed = {"fix64": True, "fix32": "fix32", "f32": False}[args.g]
    settle = settle_default(wl) if args.settle is None else args.settle

    # N > 1: the library's own NCCL exchange (bp_network_step runs the whole
    # step, the bit-packed all-gather included); --dist-backend gloo: the
    # caller-driven exchange through torch.distributed (functional check of
    # several ranks sharing one GPU)
    exchange = "nccl" if (world > 1 and args.dist_backend == "nccl") else "caller"
    exchange_note = None
    if exchange == "nccl":
        # every rank must agree before the collective create: fall back to the
        # torch.distributed exchange when any rank cannot load NCCL itself
        import paper_2311_05106_b200 as bp
        ok = torch.tensor([1 if bp.nccl_version() is not None else 0], device=dev)
        dist.all_reduce(ok, op=dist.ReduceOp.MIN)
        if int(ok.item()) == 0:
            exchange, exchange_note = "caller", "library NCCL unavailable on a rank"
    net, csr = build_network(wl, world, rank, fixed, dev, exchange=exchange)
    n_local = net.part.col_end - net.part.col_begin
    small = world == 1 and n_total <= 4096
    stream = torch.cuda.current_stream()

    def steps(k):
        if world == 1 or exchange == "nccl":
            net.run(k)
            return
        for _ in range(k):
            net.step_distributed()

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(device_index) as clk:
        # settle + warm-up (untimed)
        steps(settle)
        steps(args.warmup)
        barrier()
        sp0, ev0, _ = net.counters()
        # timed region: exactly K steps, CUDA events on the launching stream
        barrier()
        clk.mark_start()
        start.record(stream)
        steps(args.steps)
        stop.record(stream)
        barrier()
        clk.mark_stop()
    ms = start.elapsed_time(stop)
    sp1, ev1, sat1 = net.counters()
    # per-kernel durations: an instrumented window of the SAME (settled)
    # regime right after the timed region, its bytes from its own event
    # counter (events are recorded between the kernels of a step, which
    # also disables their programmatic-launch overlap: slightly slower)
    prof = None
    if world == 1 or exchange == "nccl":
        k_prof = max(args.steps, 200)
        pw0 = net.counters()
        net.net.profile_begin(k_prof)
        steps(k_prof)
        sc_ms, up_ms, nrec = net.net.profile_end()
        pw1 = net.counters()
        prof = dict(scatter_ms=sc_ms, update_ms=up_ms, steps=nrec,
                    events=pw1[1] - pw0[1], spikes=pw1[0] - pw0[0])
    events_local = ev1 - ev0
    spikes_seen = sp1 - sp0
    if world > 1:
        rdev = dev if args.dist_backend == "nccl" else "cpu"
        t = torch.tensor([ms], dtype=torch.float64, device=rdev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        e = torch.tensor([events_local], dtype=torch.float64, device=rdev)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        events_total = float(e.item())
    else:
        events_total = float(events_local)
    secs = ms / 1e3
    value = events_total / secs
    sim_ratio = args.steps * DT_MS * 1e-3 / secs

    # end-to-end through the public API with host buffers (same network, same
    # settled regime): the current state is snapshotted to pinned host memory
    # (untimed); the timed region copies it back H2D, runs the K steps and
    # reads every step's spike count D2H into pinned memory.
    e2e = None
    if not args.no_e2e and (world == 1 or exchange == "nccl"):
        e2e = run_e2e(args, net, world, dev)

    # per-rank kernel times (N > 1: every rank's window, gathered to rank 0)
    mine = None
    if prof is not None:
        nr = max(prof["steps"], 1)
        mine = {"rank": rank, "k_step_us": prof["update_ms"] * 1e3 / nr,
                "k_bin_us": prof["scatter_ms"] * 1e3 / nr, "events_per_step": prof["events"] / nr}
    per_rank = [mine]
    if world > 1:
        per_rank = [None] * world
        dist.all_gather_object(per_rank, mine)
    if rank != 0:
        if world > 1:
            dist.barrier()
            net.net.close()            # NCCL communicator destroyed while every rank is alive
            dist.barrier()
            dist.destroy_process_group()
        return

    peaks, peak_kind = _peaks()
    roofline = None
    if prof is not None:
        nrec = max(prof["steps"], 1)
        upd_s = prof["update_ms"] / 1e3 / nrec
        bin_s = prof["scatter_ms"] / 1e3 / nrec
        single = launches_per_step(spec["model"], n_local, n_total, world) == 1
        if single and world == 1:
            # one kernel per step (the dense HH update delivers its own
            # spikes): the instrumented window's per-step events block the
            # programmatic launch overlap and add launch latency, so the
            # timed region's step time is the tighter bound on the kernel
            upd_s = min(upd_s, ms / 1e3 / args.steps)
        ev_step = prof["events"] / nrec
        bytes_per_launch = state_bytes_per_neuron(spec["model"], fixed) * n_local + 4 * ev_step
        achieved = bytes_per_launch / upd_s / 1e9
        if small:
            kname = "k_small_net<%s,%s> (whole time loop in one CTA, state in shared memory)" % (
                spec["model"].upper(), args.g)
        elif spec["model"] == "hh":
            kname = ("k_hh_dense1<%s> (per-neuron event counts -> Expon+COBA+HH -> spike bits; "
                     "delivers its own spikes' events as REDs on the next step's counts)" % args.g)
        else:
            kname = ("k_step<LIF,%s> (fused: bucket counts -> Expon+COBA+LIF -> spike bits + "
                     "active list)" % args.g)
        traffic, tsrc = _ncu_traffic_r02(wl, args.g, "k_step")
        roofline = {"kernel": kname, "bound": "hbm", "achieved": achieved,
                    "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                    "traffic": traffic,
                    "traffic_source": (tsrc + " (ncu --set full of this workload after the "
                                       "settle steps; dram bytes read + write per launch)")
                    if traffic else None,
                    "peak_source": peak_kind,
                    "algorithmic_bytes_per_launch": bytes_per_launch,
                    "bytes_model": "%.3f B/neuron x %d neurons + 4 B x %.0f event records" % (
                        state_bytes_per_neuron(spec["model"], fixed), n_local, ev_step),
                    "avg_launch_us": upd_s * 1e6,
                    "share_of_step": upd_s / (upd_s + bin_s) if (upd_s + bin_s) else None,
                    "window": ("instrumented %d steps right after the timed region (same settled "
                               "regime); bytes from that window's own event counter (%.0f events "
                               "per step)" % (nrec, ev_step)) + (
                        "; kernel time = the timed region's step time (single-kernel step)"
                        if single and world == 1 else "")}
        if world > 1:
            sb = state_bytes_per_neuron(spec["model"], fixed) * n_local
            roofline["per_rank"] = [
                dict(r, frac=(sb + 4 * r["events_per_step"]) / (r["k_step_us"] * 1e-6) / 1e9 /
                     peaks["hbm_gbs"]) for r in per_rank if r]
            roofline["window"] += ("; k_step = the neuron-update kernel, k_bin = local binning "
                                   "(+ the remote scatter of the previous step for delay >= 2)")
        if small:
            roofline["note"] = ("latency-bound: the whole state (%d neurons) lives in one SM's "
                                "shared memory; HBM fraction is not the limiter" % n_local)
        elif spec["model"] == "hh":
            roofline["note"] = ("compute-latency-bound: a ~490-instruction dependent fp32 chain "
                                "per neuron (exponential Euler, 6 rate functions), one neuron per "
                                "thread; the %.1f MB of state is L2-resident, so the HBM fraction "
                                "is not the limiter" % (
                                    state_bytes_per_neuron("hh", fixed) * n_local / 1e6))
        elif spec["conn"] == "jit":
            sm_mhz = clk.summary().get("sm_mhz") or 1965.0
            peak_ops = 148 * 4 * 32 * sm_mhz * 1e6
            ops = BIN_CORE_OPS_PER_EVENT * ev_step / bin_s
            roofline["bin_kernel"] = {
                "kernel": "k_bin_sorted (regenerate JIT rows of spikes_n, stage, sort by "
                          "tile, write bucket runs)",
                "bound": "alu", "achieved": ops / 1e12, "peak": peak_ops / 1e12,
                "unit": "T lane-instructions/s", "frac": ops / peak_ops,
                "avg_launch_us": bin_s * 1e6, "events_per_launch": ev_step,
                "ops_per_event": BIN_CORE_OPS_PER_EVENT,
                "ops_source": "measured lane instructions per U[1,K] gap of k_jit_rows "
                              "(profiles/r01/ncu_gap_samplers.json): the regeneration core",
                "peak_source": "derived: 148 SMs x 4 schedulers x 32 lanes x sampled SM clock"}
    cpu = cpu_baseline(wl, n_total, csr) if (world == 1 and not args.no_cpu) else None
    state_mb = state_bytes_per_neuron(spec["model"], fixed) * n_local / 1e6
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
        "higher_is_better": True, "scaling": spec["scaling"], "vs_baseline": None,
        "dtype": {"fix64": "i64fix+f32", "fix32": "i32fix+f32", "f32": "f32"}[args.g],
        "data": "synthetic",
        "config": {"workload": wl, "description": spec["cfg"], "n_total": n_total,
                   "n_per_gpu": n_local, "model": spec["model"], "connectivity": spec["conn"],
                   "fan_in": round(net_params(wl, n_total)[0] * n_total, 3),
                   "p": net_params(wl, n_total)[0],
                   "w_exc_inh": list(net_params(wl, n_total)[1:]), "dt_ms": DT_MS,
                   "settle_steps": settle,
                   "g": {"fix64": "int64 fixed point 2^-32 (rule F1)",
                         "fix32": "int32 fixed point 2^-%d (rule F2), saturations: %d" % (
                             20 if spec["model"] == "lif" else 16, sat1),
                         "f32": "fp32, increments fl32(count*w) (rule N1-f32), bit-exact vs oracle"}[args.g],
                   "parallelism": f"postsynaptic partition x{world}",
                   "host_loop": ("library time loop (bp_network_step)" if world == 1 else
                                 "library time loop with its own NCCL spike all-gather "
                                 "(bp_network_step, BP_EXCHANGE_NCCL)" if exchange == "nccl"
                                 else "torch.distributed exchange, eager per-step calls"),
                   "seg_len": seg_len_of(wl, n_total) if spec["conn"] == "jit" else None,
                   "exchange": {"nccl": "ncclAllGather of the bit-packed local words "
                                        "(%d B per rank per step), in place, on the "
                                        "library's comm stream" % (net.part.local_words * 4),
                                "caller": "none (one GPU)" if world == 1 else
                                          "torch.distributed all_gather_into_tensor" + (
                                              " (%s)" % exchange_note if exchange_note
                                              else "")}[exchange],
                   "l2": (f"state {state_mb:.0f} MB/GPU > 2 x 126 MB L2: no flush needed"
                          if state_mb > 252 else
                          f"state {state_mb:.1f} MB is L2/SM-resident by design (the workload is that small)"),
                   "spikes": spikes_seen, "events": events_total},
        "sim_s_per_wall_s": sim_ratio,
        "events_per_step": events_total / args.steps,
        # libbp kernels in the timed region (launches_per_step; NCCL's
        # all-gather kernel not counted)
        "gpu_launches": (1 if small else
                         launches_per_step(spec["model"], n_local, n_total, world) * args.steps),
        "clocks": clocks,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": e2e,
    }
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.barrier()
        net.net.close()
        dist.barrier()
        dist.destroy_process_group()


def run_e2e(args, net, world, dev):
    """Same metric through the public API with host buffers, on the same
    (settled) network: its state is copied to pinned host memory outside the
    timed region; inside it, the state goes back H2D, the K steps run through
    bp_network_step (the NCCL exchange included for N > 1) and every step's
    spike count comes back D2H (pinned).  N > 1: max time over ranks, events
    summed."""
    import torch
    import torch.distributed as dist

    host = {k: v.to("cpu").pin_memory() for k, v in net.state.items()
            if isinstance(v, torch.Tensor)}
    counts = torch.zeros(args.steps, dtype=torch.int32).pin_memory()
    h2d = sum(t.numel() * t.element_size() for t in host.values())
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()
    sp0, ev0, _ = net.counters()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    start.record(stream)
    for k, t in host.items():
        net.state[k].copy_(t, non_blocking=True)
    net.run(args.steps, counts=counts)
    stop.record(stream)
    stop.synchronize()
    ms = start.elapsed_time(stop)
    sp1, ev1, sat1 = net.counters()
    ev = float(ev1 - ev0)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e = torch.tensor([ev], dtype=torch.float64, device=dev)
        dist.all_reduce(e, op=dist.ReduceOp.SUM)
        ms, ev = float(t.item()), float(e.item())
    return {"value": ev / (ms / 1e3), "unit": UNIT,
            "h2d_bytes_per_step": h2d / args.steps, "d2h_bytes_per_step": 4,
            "note": "settled state H2D (pinned) amortised over the K steps; per-step "
                    "spike count D2H into pinned memory; %sms=%.3f" % (
                        "per rank, max over ranks; " if world > 1 else "", ms),
            "spikes_total": int(counts.sum().item())}


def run_emulated_rank(args):
    """One rank of a G-GPU weak-scaling run, on one GPU: rank 0's partition
    (12.5 M neurons) of the G x 12.5 M network steps with scatter (remote
    rows regenerated restricted to the local segment) + update (fold, LIF,
    local binning), and the all-gather is replaced by one device copy that
    replicates rank 0's own spike words into every remote slot (the bytes
    NCCL would write; the remote ranks then fire like rank 0, which keeps
    the E/I feedback of the network -- fixed synthetic remote rates do not:
    they let rank 0's excitatory neurons run away).  Not a multi-GPU number:
    the per-rank compute of one (no NVLink in it)."""
    import torch

    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)
    G = args.emulate_world
    wl = args.workload
    n = network_size(wl, G)
    R = args.emulate_rank
    net, _ = build_network(wl, G, R, {"fix64": True, "fix32": "fix32", "f32": False}[args.g],
                           torch.device("cuda", 0))
    lw = net.part.local_words
    words = net.spikes.numel()
    assert words == G * lw
    slots = net.spikes.view(G, lw)
    local = slots[R].clone()

    comm = torch.cuda.Stream(device=0)

    def step(k):
        net.net.scatter()
        if args.emu_serial:
            net.net.update()
            # every slot <- this rank's words (its own slot: the same values)
            local.copy_(slots[R])
            slots.copy_(local.expand(G, lw))
            return
        # as CobaNetwork.step_distributed(overlap=True): the exchange stream
        # waits for this step's spike words only, so the stand-in all-gather
        # overlaps the local binning, and the next scatter waits for it
        compute = torch.cuda.current_stream(0)      # (the capture stream inside a graph)
        net.net.update_overlap(comm)
        with torch.cuda.stream(comm):
            local.copy_(slots[R])
            slots.copy_(local.expand(G, lw))
        compute.wait_stream(comm)

    settle = settle_default(wl) if args.settle is None else args.settle
    for k in range(settle + args.warmup):
        step(k)
    torch.cuda.synchronize()
    # one period of steps in a CUDA graph, as the N > 1 bench replays it
    period = math.lcm(2, net.delay + 1)
    graph = None
    if not args.no_graph:
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for k in range(period):
                step(k)
        graph.replay()
        torch.cuda.synchronize()
    sp0, ev0, _ = net.counters()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(0) as clk:
        clk.mark_start()
        a.record()
        if graph is not None:
            for _ in range(args.steps // period):
                graph.replay()
            for k in range(args.steps % period):
                step(k)
        else:
            for k in range(args.steps):
                step(k)
        b.record()
        torch.cuda.synchronize()
        clk.mark_stop()
    ms = a.elapsed_time(b)
    sp1, ev1, _ = net.counters()
    line = {"metric": METRIC + " (emulated single rank)", "value": (ev1 - ev0) / (ms / 1e3),
            "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": args.g, "data": "synthetic",
            "config": {"workload": "%s rank %d of %d" % (wl, R, G), "n_total": n,
                       "n_per_gpu": net.part.col_end - net.part.col_begin, "emulated_world": G,
                       "exchange": "replaced by a device copy of this rank's spike words "
                                   "into the %d remote slots (%.1f MB/step), %s" % (
                                       G - 1, (words - lw) * 4 / 1e6,
                                       "after the local binning (serial)" if args.emu_serial
                                       else "on an exchange stream overlapping the local "
                                            "binning (CobaNetwork.step_distributed's schedule)"),
                       "host_loop": "CUDA graph of %d steps" % period if graph is not None
                                    else "eager",
                       "settle_steps": settle,
                       "local_spikes_per_step": (sp1 - sp0) / args.steps,
                       "events_per_step": (ev1 - ev0) / args.steps},
            "clocks": clk.summary()}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# config 2: event_csrmv / jitconn event_mv microbenchmark, 100k x 100k
# ---------------------------------------------------------------------------
# Algorithmic integer ops per JIT event (homo law): Philox4x32-10 = 10 rounds
# x (2 IMAD.WIDE + 2 LOP3 + 2 key IADD) = 60 ops per 4 gap words -> 15;
# bounded draw 2; running position 1; share of the 5-step warp scan 2.5;
# RED 1.  Uniform adds 15 + 2 (weight word + fma), normal 30 + ~40 (fp64
# log/cos/sqrt, counted as 40).  Issue peak: 148 SMs x 4 schedulers x 32
# lanes x 1 warp-instruction per cycle at the sampled SM clock.
JIT_OPS_PER_EVENT = {"homo": 21.5, "uniform": 38.5, "normal": 91.5}
# Per gap draw, MEASURED: ncu smsp__inst_executed x 32 lanes / gaps of one
# k_jit_rows call (100 k x 100 k, p = 0.05; profiles/r01/ncu_gap_samplers.json):
# the paper's U[1, K] gaps (rule J3) 27.4 lane instructions, Geo(p) by
# inversion with the specified log (rule J10) 86.8.
JIT_OPS_PER_GAP = {"uniform": 27.4, "geometric": 86.8}


def run_micro(args):
    import numpy as np
    import torch

    import __graft_entry__ as ge
    ge.build_lib()
    import paper_2311_05106_b200 as bp
    from paper_2311_05106_b200 import inputs

    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    n = 100_000
    p, d, kind = args.p, args.density, args.workload
    fixed = args.fix
    law = args.law
    n_pat = 64
    pats = [inputs.spike_pattern(n, d, 7000 + k) for k in range(n_pat)]
    spikes = [torch.from_numpy(inputs.pack_bits(e).view(np.int32)).to(dev) for e in pats]
    out = torch.zeros(n, dtype=torch.int64 if fixed else torch.float32, device=dev)
    ws_bytes = (bp.lib().bp_csrmv_workspace_bytes(n, n, 1 if fixed else 0) if kind == "csrmv"
                else bp.lib().bp_jitconn_workspace_bytes(n, 0, n, 1 if fixed else 0))
    ws = torch.empty(ws_bytes, dtype=torch.uint8, device=dev)
    seed = 0xBE7C4
    geo = args.gap == "geometric"
    spec = bp.jitconn_spec(seed, p, gap_law=bp.GAP_GEOMETRIC if geo else bp.GAP_UNIFORM)
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-0.1, 0.1),
              "normal": (0.0, 1.0 / np.sqrt(n * p))}[law]     # Table S1 scales
    if kind == "csrmv":
        ip, ix, dat = bp.jitconn_materialize(spec, n, n, law=bp.LAW_UNIFORM, w0=-0.1, w1=0.1,
                                             with_data=(law != "homo"), device=dev)
        row_nnz = (ip[1:] - ip[:-1]).cpu().numpy()
        data = dat if law != "homo" else None
        # the matrix is fixed across calls: split points analysed once,
        # outside the timed region (like the CSR itself); --no-plan: per call
        plan = None if args.no_plan else bp.csrmv_plan(ip, ix, n, n, out.dtype, homo=data is None, data=data)
        call = lambda s: bp.event_csrmv(ip, ix, data, 0.6, n, n, s, out, ws=ws, plan=plan)
        ev_per_pat = [int(row_nnz[e.astype(bool)].sum()) for e in pats]
        bytes_per_event = 8 if law != "homo" else 4
        nnz = int(ip[-1].item())
        working_set = nnz * bytes_per_event + ip.numel() * 8
    elif kind == "jitrows":
        # gap-sampler cost (App. C; NEXT 4): regenerate every row
        # of the matrix (bp_jitconn_row_counts: gap chains only, no weights,
        # no scatter) -- one call = n_rows x fan-out gap draws
        counts = torch.empty(n, dtype=torch.int64, device=dev)
        c_spec = bp._binding.ctypes.byref(spec)

        def call(_s):
            bp._binding._check(bp.lib().bp_jitconn_row_counts(
                c_spec, n, n, bp._binding._ptr(counts), bp._binding._stream()))
        call(None)
        torch.cuda.synchronize()
        ev_per_pat = [int(counts.sum().item())] * n_pat
        working_set = n * 8
    else:
        fn = {"homo": bp.jitconn_event_mv_homo, "uniform": bp.jitconn_event_mv_uniform,
              "normal": bp.jitconn_event_mv_normal}[law]
        if kind == "jitmv_vec":
            # non-event mv_prob_* (NEXT 1): a float vector whose non-zeros sit
            # on the same Bernoulli patterns (density = fraction of non-zeros)
            code = {"homo": bp.LAW_HOMO, "uniform": bp.LAW_UNIFORM, "normal": bp.LAW_NORMAL}[law]
            rng = np.random.default_rng(11)
            spikes = [torch.from_numpy((e * rng.normal(0.0, 1.0, n)).astype(np.float32)).to(dev)
                      for e in pats]
            call = lambda vv: bp.jitconn_mv(code, spec, w0, w1, vv, n, n, out, ws=ws)
        elif law == "homo":
            call = lambda s: fn(spec, w0, s, n, n, out, ws=ws)
        else:
            call = lambda s: fn(spec, w0, w1, s, n, n, out, ws=ws)
        counts = torch.empty(n, dtype=torch.int64, device=dev)
        bp.lib().bp_jitconn_row_counts(bp._binding.ctypes.byref(spec), n, n,
                                       bp._binding._ptr(counts), bp._binding._stream())
        torch.cuda.synchronize()
        row_nnz = counts.cpu().numpy()
        ev_per_pat = [int(row_nnz[e.astype(bool)].sum()) for e in pats]
        working_set = n * out.element_size()
    l2 = 126 * 2 ** 20
    flush = working_set < 2 * l2
    scratch = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev) if flush else None
    stream = torch.cuda.current_stream()
    for k in range(args.warmup):
        call(spikes[k % n_pat])
    torch.cuda.synchronize()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
           for _ in range(args.steps)]
    with ClockSampler(0) as clk:
        clk.mark_start()
        for k in range(args.steps):
            if flush:
                scratch.fill_(k & 0xFF)           # evict the working set from L2
            evs[k][0].record(stream)
            call(spikes[k % n_pat])
            evs[k][1].record(stream)
        torch.cuda.synchronize()
        clk.mark_stop()
    ms = [a.elapsed_time(b) for a, b in evs]
    total_ms = sum(ms)
    events = sum(ev_per_pat[k % n_pat] for k in range(args.steps))
    value = events / (total_ms / 1e3)
    peaks, peak_kind = _peaks()
    clocks = clk.summary()
    active = sum(int(pats[k % n_pat].sum()) for k in range(args.steps)) / args.steps
    if kind == "csrmv":
        per_call = (events / args.steps) * bytes_per_event + 16 * active + n / 8 + \
            n * out.element_size()
        achieved = per_call / (total_ms / args.steps / 1e3) / 1e9
        roof = {"kernel": "k_compact + k_csr_stream (split plan precomputed)" if not args.no_plan
                else "k_compact + k_csr_split + k_csr_stream", "bound": "hbm", "achieved": achieved,
                "peak": peaks["hbm_gbs"], "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"],
                "traffic": None, "peak_source": peak_kind,
                "algorithmic_bytes_per_launch": per_call}
    else:
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        peak_ops = 148 * 4 * 32 * sm_mhz * 1e6
        ops_ev = (JIT_OPS_PER_GAP[args.gap] if kind == "jitrows"
                  else JIT_OPS_PER_EVENT[law] + (JIT_OPS_PER_GAP["geometric"] -
                                                 JIT_OPS_PER_GAP["uniform"]) * geo)
        ops = ops_ev * events / (total_ms / 1e3)
        kern = ("k_jit_rows (row counts: gap chains only)" if kind == "jitrows" else
                "%sk_jit_tiled<%s> (k_jit_scatter for rows < 1000 events, normal law)"
                % ("" if kind == "jitmv_vec" else "k_compact + ", law))
        roof = {"kernel": kern, "bound": "alu",
                "achieved": ops / 1e12, "peak": peak_ops / 1e12, "unit": "Tops/s (int32 lane ops)",
                "frac": ops / peak_ops, "traffic": None,
                "peak_source": "derived: 148 SMs x 4 schedulers x 32 lanes x sampled SM clock",
                "ops_per_event": ops_ev}
    line = {"metric": "synaptic events/sec (event_mv microbenchmark, config 2)",
            "value": value, "unit": UNIT, "n_gpus": 1, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps,
            "higher_is_better": True, "scaling": "none", "vs_baseline": None,
            "dtype": "i64fix" if fixed else "f32", "data": "synthetic",
            "config": {"workload": f"{kind}_{law}" + ("_geo" if geo else ""), "shape": [n, n],
                       "p": p, "density": d, "gap_sampler": args.gap,
                       "K": bp.conn_len(p), "events_per_call": events / args.steps,
                       "active_rows_per_call": active,
                       "csr_plan": (kind == "csrmv" and not args.no_plan),
                       "l2": ("flushed between calls (256 MB write)" if flush
                              else "working set %.0f MB > 2 x L2" % (working_set / 1e6))},
            # compact + scatter (+ per-call split of the rows without a plan)
            "gpu_launches": {"csrmv": 3 if args.no_plan else 2, "jitmv": 2, "jitmv_vec": 1,
                             "jitrows": 1}[kind] * args.steps,
            "clocks": clocks, "roofline": roof,
            "call_us": {"median": float(np.median(ms)) * 1e3, "min": float(np.min(ms)) * 1e3}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# Fig 3A/B: memory and speed of the JIT operator
# y = J v against the same matrix materialised, as n grows at fixed p
# ---------------------------------------------------------------------------
def _time_calls(fn, reps, flush=None):
    """Median device time of `reps` calls (CUDA events on the current stream;
    the L2 scratch write between calls when `flush` is given)."""
    import torch
    st = torch.cuda.current_stream()
    fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        fn()
        b.record(st)
        b.synchronize()
        ts.append(a.elapsed_time(b))
    return statistics.median(ts) * 1e3


def run_fig3ab(args):
    """For n in a sweep (square n x n, connection probability p, normal
    weights N(0, 1/(n p)), the Table S1 scale), one JSON line per n:
      * device bytes the connectivity occupies: JIT = 0 (four scalars,
        P:192), CSR = indptr + indices + weights, dense = 4 n^2;
      * time per call of the non-event product y = J v (v dense, fp32) --
        bp_jitconn_mv_normal (ours) vs the same matrix materialised by the
        library's own generator and multiplied by cuSPARSE SpMV
        (torch.sparse_csr) and, while 4 n^2 fits the budget, dense cuBLAS
        (torch.mv) -- the comparison systems of Fig 3A/B as library calls;
      * time per call of the event-driven product at 10 % spike density:
        bp_jitconn_event_mv_normal vs bp_event_csrmv on the materialised
        matrix (both ours).
    Matrices over --fig3-budget-gb of device memory are skipped (reported)."""
    import numpy as np
    import torch

    import __graft_entry__ as ge
    ge.build_lib()
    import paper_2311_05106_b200 as bp
    from paper_2311_05106_b200 import inputs
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    p = args.p
    budget = args.fig3_budget_gb * 1e9
    flush = torch.empty(256 * 2 ** 20, dtype=torch.uint8, device=dev)
    sizes = [int(x) for x in args.fig3_sizes.split(",")]
    for n in sizes:
        seed = 0xF163
        spec = bp.jitconn_spec(seed, p)
        mu, sigma = 0.0, 1.0 / math.sqrt(n * p)
        rng = np.random.default_rng(5)
        v = torch.from_numpy(rng.standard_normal(n).astype(np.float32)).to(dev)
        ev = inputs.spike_pattern(n, 0.1, 9000 + n % 1000)
        spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).to(dev)
        out = torch.zeros(n, dtype=torch.float32, device=dev)
        ws = torch.empty(bp.lib().bp_jitconn_workspace_bytes(n, 0, n, 0), dtype=torch.uint8,
                         device=dev)
        reps = max(3, min(args.steps, int(2e10 / max(n * n * p, 1.0))))
        rec = {"workload": "fig3ab", "n": n, "p": p, "K": bp.conn_len(p),
               "weights": "normal(0, 1/(n p))", "expected_nnz": n * n * 2.0 / (bp.conn_len(p) + 1),
               "reps": reps}
        rec["jit_bytes"] = 0
        rec["jit_mv_us"] = _time_calls(lambda: bp.jitconn_mv(bp.LAW_NORMAL, spec, mu, sigma, v, n,
                                                             n, out, ws=ws), reps, flush)
        rec["jit_event_mv_us"] = _time_calls(lambda: bp.jitconn_event_mv_normal(
            spec, mu, sigma, spikes, n, n, out, ws=ws), reps, flush)
        csr_bytes = 8 * (n + 1) + 8 * rec["expected_nnz"]
        rec["csr_bytes"] = csr_bytes
        if csr_bytes <= budget:
            ip, ix, dat = bp.jitconn_materialize(spec, n, n, law=bp.LAW_NORMAL, w0=mu, w1=sigma,
                                                 device=dev)
            nnz = int(ix.numel())
            rec["nnz"] = nnz
            rec["csr_bytes"] = ip.numel() * 8 + nnz * 8
            # the materialised matrix IS the JIT matrix: one call of each agrees
            bp.jitconn_mv(bp.LAW_NORMAL, spec, mu, sigma, v, n, n, out, ws=ws)
            y_jit = out.clone()
            A = torch.sparse_csr_tensor(ip, ix, dat, size=(n, n))
            # Listing S2 scatters rows into columns: y = J^T v with J rows = pre
            At = A.t().to_sparse_csr()
            y_sp = torch.mv(At, v)
            err = (y_sp - y_jit).abs().max().item()
            scale = torch.mv(At.abs() if hasattr(At, "abs") else At, v.abs()).max().item()
            rec["jit_vs_cusparse_max_abs_diff"] = err
            rec["jit_vs_cusparse_rel_to_sum_abs"] = err / max(scale, 1e-30)
            rec["cusparse_spmv_us"] = _time_calls(lambda: torch.mv(At, v), reps, flush)
            del A
            cws = torch.empty(bp.lib().bp_csrmv_workspace_bytes(n, n, 0), dtype=torch.uint8,
                              device=dev)
            plan = bp.csrmv_plan(ip, ix, n, n, torch.float32, homo=False, data=dat)
            rec["csr_event_mv_us"] = _time_calls(lambda: bp.event_csrmv(
                ip, ix, dat, 0.0, n, n, spikes, out, ws=cws, plan=plan), reps, flush)
            del At, ip, ix, dat, plan, cws
        else:
            rec["csr_skipped"] = "CSR would need %.1f GB > budget" % (csr_bytes / 1e9)
        dense_bytes = 4.0 * n * n
        rec["dense_bytes"] = dense_bytes
        if dense_bytes <= budget and n <= 150_000:
            D = torch.zeros((n, n), dtype=torch.float32, device=dev)
            ipd, ixd, datd = bp.jitconn_materialize(spec, n, n, law=bp.LAW_NORMAL, w0=mu,
                                                    w1=sigma, device=dev)
            rows = torch.repeat_interleave(torch.arange(n, device=dev), ipd[1:] - ipd[:-1])
            D[ixd.long(), rows] = datd            # D = J^T (column r = row r of J)
            del ipd, ixd, datd, rows
            rec["dense_mv_us"] = _time_calls(lambda: torch.mv(D, v), reps, flush)
            del D
        else:
            rec["dense_skipped"] = "dense would need %.1f GB" % (dense_bytes / 1e9)
        torch.cuda.empty_cache()
        print(json.dumps(rec), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10_000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--g", choices=["fix64", "fix32", "f32"], default="f32",
                    help="conductance representation: int64 2^-32 (rule F1), int32 "
                         "2^-F (rule F2) or fp32 (rule T3 parity)")
    ap.add_argument("--f32", action="store_true", help="alias of --g f32")
    ap.add_argument("--no-cpu", action="store_true", help="skip the cpu_baseline leg")
    ap.add_argument("--settle", type=int, default=None,
                    help="untimed pre-roll steps before the warm-up (default: 2000 for "
                         "networks > 4096 neurons, the initial synchronous burst)")
    ap.add_argument("--no-e2e", action="store_true", help="skip the host-buffer e2e leg")
    ap.add_argument("--emulate-world", type=int, default=0,
                    help="one GPU: time rank 0 of a G-GPU weak-scaling run (exchange "
                         "replaced by a device copy; not a multi-GPU number)")
    ap.add_argument("--emulate-rank", type=int, default=0,
                    help="--emulate-world: which rank's partition to time")
    ap.add_argument("--emu-serial", action="store_true",
                    help="--emulate-world: the stand-in exchange after the local binning "
                         "instead of overlapping it")
    ap.add_argument("--no-graph", action="store_true",
                    help="--emulate-world: eager per-step calls instead of a CUDA graph")
    ap.add_argument("--fig3-sizes", default="10000,30000,100000,300000,1000000,3000000",
                    help="--workload fig3ab: matrix sizes n")
    ap.add_argument("--fig3-budget-gb", type=float, default=60.0,
                    help="--workload fig3ab: largest materialised matrix")
    ap.add_argument("--workload",
                    choices=list(NETWORKS) + ["csrmv", "jitmv", "jitmv_vec", "jitrows", "fig3ab"],
                    default="coba_lif_jit")
    ap.add_argument("--p", type=float, default=0.05, help="microbench connection probability")
    ap.add_argument("--density", type=float, default=0.1, help="microbench spike density")
    ap.add_argument("--law", choices=["homo", "uniform", "normal"], default="uniform")
    ap.add_argument("--fix", action="store_true", help="microbench int64 fixed-point output")
    ap.add_argument("--gap", choices=["uniform", "geometric"], default="uniform",
                    help="JIT gap sampler: the paper's U[1, K] (rule J3) or Geo(p) "
                         "by inversion (rule J10, P:340)")
    ap.add_argument("--no-plan", action="store_true",
                    help="csrmv microbench: split rows on every call (no csrmv_plan)")
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="spike exchange backend for --gpus > 1 (gloo: functional check "
                         "with several ranks on one GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.f32:
        args.g = "f32"
    if args.gpus > 1 and "RANK" not in os.environ and args.impl == "ours" \
            and args.emulate_world <= 1:
        # `python bench.py --gpus N`: launch the N ranks ourselves (one per
        # GPU), exactly as the driver's torchrun command does
        import socket
        with socket.socket() as sk:
            sk.bind(("127.0.0.1", 0))
            port = sk.getsockname()[1]
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
                                  f"--master-port={port}", os.path.abspath(__file__),
                                  *sys.argv[1:]])
    if args.impl == "reference":
        run_reference(args)
    elif args.emulate_world > 1:
        run_emulated_rank(args)
    elif args.workload == "fig3ab":
        run_fig3ab(args)
    elif args.workload in ("csrmv", "jitmv", "jitmv_vec", "jitrows"):
        run_micro(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
