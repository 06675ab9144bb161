"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the oracle computes these in seconds to minutes because its work is
event-driven; its order-free loops use every host core, bit-identical to
one thread):

* config 5 / bench default: the 12.5M-neuron COBA-LIF JIT network, first
  steps of the run (step 0 spikes ~0.6 % of the neurons, so step 1 delivers
  ~6 M synaptic events), every conductance mode, compared bit for bit; and
  300 steps in the f32 (bench) and fix32 modes -- the synchronous burst
  (up to 435 k spikes = 35 M events per step) and the settled regime after
  it (~25 k spikes per step from step ~150 on);
* config 4: the 400k-neuron COBA-HH CSR network, 100 steps, all three modes;
* config 2: the 100k x 100k event_csrmv / jitconn event_mv cells, including
  the CSR p = 0.05 / 10 % heterogeneous cell the bench judges.
"""
import os

import numpy as np
import pytest
import torch

from paper_2311_05106_b200 import inputs
from paper_2311_05106_b200.network import SEED_E, SEED_I, CobaNetwork

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)


@pytest.mark.parametrize("mode", ["f32", "fix32", "fix64"])
def test_config5_network_first_steps(orc, mode):
    n, steps = 12_500_000, 3
    net = CobaNetwork(n, conn="jit", fixed={"f32": False, "fix32": "fix32", "fix64": True}[mode])
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    got = raster.cpu().numpy().view(np.uint32)
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, n, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, n, orc.LAW_HOMO, 6.7))
    g = {"f32": np.float32, "fix32": np.int32, "fix64": np.int64}[mode]
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, g), g_i=np.zeros(n, g),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want[0].sum() > 50_000                  # the step-0 burst
    for k in range(steps):
        assert np.array_equal(got[k], inputs.pack_bits(want[k])), k
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
    assert np.array_equal(net.state["g_e"].cpu().numpy(), st["g_e"])
    assert np.array_equal(net.state["g_i"].cpu().numpy(), st["g_i"])


@pytest.mark.timeout(900)
def test_1e8_neurons_on_one_gpu_first_steps(orc):
    """The north_star's >= 1e8-neuron COBA-LIF JIT network (config 5's total
    size) fits one B200: its first steps (step 0 spikes ~0.6 % = ~600 k
    neurons, so step 1 delivers ~48 M synaptic events) bit for bit."""
    n, steps = 100_000_000, 2
    net = CobaNetwork(n, conn="jit", fixed=False)
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    got = raster.cpu().numpy().view(np.uint32)
    v_gpu = net.state["v"].cpu().numpy()
    ge_gpu = net.state["g_e"].cpu().numpy()
    del net
    torch.cuda.empty_cache()
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    assert K == n // 40 - 1
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, n, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, n, orc.LAW_HOMO, 6.7))
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.float32), g_i=np.zeros(n, np.float32),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want[0].sum() > 400_000
    for k in range(steps):
        assert np.array_equal(got[k], inputs.pack_bits(want[k])), k
    assert np.array_equal(v_gpu.view(np.uint32), st["v"].view(np.uint32))
    assert np.array_equal(ge_gpu.view(np.uint32), st["g_e"].view(np.uint32))


def test_config2_csr_full_size(bp, orc):
    n, p, d = 100_000, 0.01, 0.1
    ip, ix, _ = inputs.fixed_fanin_csr_fast(n, n, p, seed=17)
    rng = np.random.default_rng(3)
    dat = rng.uniform(-0.1, 0.1, ix.shape[0]).astype(np.float32)
    ev = inputs.spike_pattern(n, d, 7000)
    spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()
    tip, tix, tdat = (torch.from_numpy(a).cuda() for a in (ip, ix, dat))
    out = torch.zeros(n, dtype=torch.int64, device="cuda")
    bp.event_csrmv(tip, tix, tdat, 0.0, n, n, spikes, out)
    want = orc.event_csrmv(ip, ix, dat, 0.0, n, n, ev, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want)
    out32 = torch.zeros(n, dtype=torch.float32, device="cuda")
    bp.event_csrmv(tip, tix, tdat, 0.0, n, n, spikes, out32)
    ref, absw = orc.event_csrmv(ip, ix, dat, 0.0, n, n, ev, orc.OUT_F64, with_abs=True)
    err = np.abs(out32.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)


@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
def test_config2_jitconn_full_size(bp, orc, law):
    n, p, d = 100_000, 0.05, 0.01
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-0.1, 0.1),
              "normal": (0.0, 1.0 / np.sqrt(n * p))}[law]
    seed = 0xBE7C4
    ev = inputs.spike_pattern(n, d, 7001)
    spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()
    spec = bp.jitconn_spec(seed, p)
    out = torch.zeros(n, dtype=torch.int64, device="cuda")
    fn = {"homo": lambda o: bp.jitconn_event_mv_homo(spec, w0, spikes, n, n, o),
          "uniform": lambda o: bp.jitconn_event_mv_uniform(spec, w0, w1, spikes, n, n, o),
          "normal": lambda o: bp.jitconn_event_mv_normal(spec, w0, w1, spikes, n, n, o)}[law]
    fn(out)
    ospec = orc.JitSpec(seed, orc.conn_len(p), n, orc.LAWS[law], w0, w1)
    want = orc.jit_event_mv(ospec, n, n, ev, out_kind=orc.OUT_FIX)
    got = out.cpu().numpy()
    assert np.array_equal(got, want)              # every law bit-exact (J7n)


@pytest.fixture(scope="module")
def bp():
    import paper_2311_05106_b200 as bp
    return bp


@pytest.fixture()
def threads(orc):
    orc.set_threads(os.cpu_count() or 1)
    yield
    orc.set_threads(1)


@pytest.mark.timeout(3000)
@pytest.mark.parametrize("mode", ["f32", "fix32"])
def test_config5_network_300_steps(orc, threads, mode):
    """Config 5 at full size (12.5 M neurons) for 300 steps: every step's
    spike words, then V, g and the refractory counters bit for bit."""
    n, steps = 12_500_000, 300
    net = CobaNetwork(n, conn="jit", fixed={"f32": False, "fix32": "fix32"}[mode])
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    got = raster.cpu().numpy().view(np.uint32)
    state_gpu = {k: v.cpu().numpy() for k, v in net.state.items() if isinstance(v, torch.Tensor)}
    del net, raster
    torch.cuda.empty_cache()
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, n, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, n, orc.LAW_HOMO, 6.7))
    g = {"f32": np.float32, "fix32": np.int32}[mode]
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, g), g_i=np.zeros(n, g),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    spikes = []
    for k in range(steps):
        row = orc.run_network("lif", orc.lif_params(), st, pe, pi, 1)[0]
        spikes.append(int(row.sum()))
        assert np.array_equal(got[k], inputs.pack_bits(row)), k
    assert max(spikes) > 300_000                     # the burst
    assert 5_000 < np.mean(spikes[-50:]) < 100_000   # the settled regime
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(state_gpu[k].view(np.uint8), st[k].view(np.uint8)), k


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("mode", ["f32", "fix32", "fix64"])
def test_config4_hh400k_100_steps(orc, threads, mode):
    """Config 4 at full size: the 400k-neuron COBA-HH network over stored
    CSR (= the oracle's materialisation of the JIT spec, fan-in 80, reading
    R25) for 100 steps, in the bench's launch configuration (dense
    delivery, k_hh_dense1), bit for bit in every conductance mode."""
    n, steps = 400_000, 100
    n_exc = n * 4 // 5
    p = 80.0 / n
    K = orc.conn_len(p)
    je = orc.JitSpec(SEED_E, K, n, orc.LAW_HOMO, 6.0)
    ji = orc.JitSpec(SEED_I, K, n, orc.LAW_HOMO, 67.0)
    ipe, ixe, _ = orc.jit_materialize(je, n_exc, n)
    ipi, ixi, _ = orc.jit_materialize(ji, n - n_exc, n)
    csr = ((torch.from_numpy(ipe).cuda(), torch.from_numpy(ixe).cuda()),
           (torch.from_numpy(ipi).cuda(), torch.from_numpy(ixi).cuda()))
    fixed = {"f32": False, "fix32": "fix32", "fix64": True}[mode]
    net = CobaNetwork(n, model="hh", conn="csr", fixed=fixed, csr=csr, p=p)
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    got = raster.cpu().numpy().view(np.uint32)
    g = {"f32": np.float32, "fix32": np.int32, "fix64": np.int64}[mode]
    orc.set_fix32_bits(16)
    v, m, h, nk = inputs.hh_init(n)
    st = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, g), g_i=np.zeros(n, g),
              spikes=np.zeros(n, np.uint8))
    pe = orc.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=6.0)
    pi = orc.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=67.0)
    want = orc.run_network("hh", orc.hh_params(), st, pe, pi, steps)
    orc.set_fix32_bits(20)
    assert want.sum() > 1000
    for k in range(steps):
        assert np.array_equal(got[k], inputs.pack_bits(want[k])), k
    for k, key in (("v", "v"), ("m", "m"), ("h", "h"), ("n", "n"), ("g_e", "g_e"),
                   ("g_i", "g_i")):
        assert np.array_equal(net.state[k].cpu().numpy().view(np.uint8),
                              st[key].view(np.uint8)), k


@pytest.mark.timeout(1200)
def test_config2_csr_p005_hetero_full_size(bp, orc):
    """The CSR cell the bench judges against the HBM roofline: 100k x 100k,
    p = 0.05 (5e8 entries, Bernoulli rows), heterogeneous U[-0.1, 0.1)
    weights, 10 % spike density, in the bench's launch configuration (split
    plan computed once) and without a plan: fix64 bit-exact, f32 within
    rule T2 per output."""
    n, p, d = 100_000, 0.05, 0.1
    ip, ix, dat = inputs.bernoulli_csr(n, n, p, seed=21, weights="uniform", w0=-0.1, w1=0.1)
    ev = inputs.spike_pattern(n, d, 7000)
    spikes = torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()
    tip, tix, tdat = (torch.from_numpy(a).cuda() for a in (ip, ix, dat))
    want = orc.event_csrmv(ip, ix, dat, 0.0, n, n, ev, orc.OUT_FIX)
    ref, absw = orc.event_csrmv(ip, ix, dat, 0.0, n, n, ev, orc.OUT_F64, with_abs=True)
    for planned in (True, False):
        out = torch.zeros(n, dtype=torch.int64, device="cuda")
        out32 = torch.zeros(n, dtype=torch.float32, device="cuda")
        for o in (out, out32):
            plan = bp.csrmv_plan(tip, tix, n, n, o.dtype, homo=False, data=tdat) if planned else None
            ws = torch.empty(bp.lib().bp_csrmv_workspace_bytes(n, n, 1 if o.dtype == torch.int64
                                                               else 0),
                             dtype=torch.uint8, device="cuda")
            bp.event_csrmv(tip, tix, tdat, 0.0, n, n, spikes, o, ws=ws, plan=plan)
        assert np.array_equal(out.cpu().numpy(), want), planned
        err = np.abs(out32.cpu().numpy().astype(np.float64) - ref)
        assert np.all(err <= 1e-5 * absw + 1e-30), planned
