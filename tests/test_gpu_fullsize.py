"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (the oracle computes these in seconds because work is event-driven):

* config 5 / bench default: the 12.5M-neuron COBA-LIF JIT network, first
  steps of the run (step 0 spikes ~0.6 % of the neurons, so step 1 delivers
  ~6 M synaptic events), every conductance mode, compared bit for bit;
* config 2: the 100k x 100k event_csrmv / jitconn event_mv cells.
"""
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
