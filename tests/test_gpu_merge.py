"""GPU parity of networks with several projections merged per receptor
(AlignPost) and of the library's
own NCCL exchange (bp_network_create with BP_EXCHANGE_NCCL),
bit for bit against the oracle's run_network.

Layouts:
* split    -- Listing S3 with the E population cut into two JIT projections
              of the same weight (different seeds): one weight class per
              receptor, the standard k_step fold;
* general  -- two E weights and two I weights (4 weight classes, the
              general merge: exact integer sums, fp32 rounded once);
* mixed    -- a CSR projection and JIT projections into the same receptor,
              3-step synaptic delay.
"""
import numpy as np
import pytest
import torch

from paper_2311_05106_b200 import inputs
from paper_2311_05106_b200.network import CobaNetwork, ProjSpec

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)


def _layout(orc, name, n):
    """(ProjSpecs for the library, oracle Projections, delay)."""
    n_exc = n * 4 // 5
    p = 80.0 / n
    K = orc.conn_len(p)
    c1 = n_exc // 3
    if name == "split":
        rows = [(0, c1, "exc", 0.6, 101), (c1, n_exc, "exc", 0.6, 102), (n_exc, n, "inh", 6.7, 103)]
        delay, csr_rows = 1, None
    elif name == "general":
        c2 = n_exc + (n - n_exc) // 2
        rows = [(0, c1, "exc", 0.6, 201), (c1, n_exc, "exc", 0.45, 202),
                (n_exc, c2, "inh", 6.7, 203), (c2, n, "inh", 5.0, 204)]
        delay, csr_rows = 1, None
    else:   # mixed: projection 0 is stored CSR
        rows = [(0, c1, "exc", 0.6, 301), (c1, n_exc, "exc", 0.5, 302), (n_exc, n, "inh", 6.7, 303)]
        delay, csr_rows = 3, 0
    specs, oproj = [], []
    for k, (b, e, rec, w, seed) in enumerate(rows):
        jit = orc.JitSpec(seed, K, n, orc.LAW_HOMO, w)
        if k == csr_rows:
            ip, ix, _ = orc.jit_materialize(jit, e - b, n)
            specs.append(ProjSpec(b, e, rec, w, csr=(torch.from_numpy(ip), torch.from_numpy(ix))))
            oproj.append(orc.Projection(b, e - b, csr=(ip, ix, None), w_homo=w, receptor=rec))
        else:
            specs.append(ProjSpec(b, e, rec, w, seed=seed, p=p))
            oproj.append(orc.Projection(b, e - b, jit=jit, receptor=rec))
    return specs, oproj, delay


def _g(mode):
    return {"fix64": np.int64, "fix32": np.int32, "f32": np.float32}[mode]


@pytest.mark.parametrize("mode", ["fix64", "fix32", "f32"])
@pytest.mark.parametrize("layout", ["split", "general", "mixed"])
@pytest.mark.parametrize("n,steps", [(4000, 600), (20_000, 300)])
def test_merged_network_bit_exact(orc, layout, mode, n, steps):
    specs, oproj, delay = _layout(orc, layout, n)
    net = CobaNetwork(n, conn="jit", fixed={"fix64": True, "fix32": "fix32", "f32": False}[mode],
                      projections=specs, delay=delay)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, _g(mode)), g_i=np.zeros(n, _g(mode)),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, oproj, None, steps, delay=delay)
    got = np.stack([inputs.unpack_bits(r, n) for r in raster.cpu().numpy().view(np.uint32)])
    assert want.sum() > 0
    assert np.array_equal(got, want)
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(net.state[k].cpu().numpy().view(np.uint8), st[k].view(np.uint8)), k


def test_merged_conductance_memory(orc):
    """The merged network holds ONE g_E and ONE g_I array whatever the number
    of projections: the state bytes are those of Listing S3's
    two-projection network, and the library's own allocation (buckets +
    projection table) grows only by the table and the extra count classes."""
    n = 100_000
    specs, _, _ = _layout(orc, "general", n)
    merged = CobaNetwork(n, conn="jit", fixed=False, projections=specs)
    plain = CobaNetwork(n, conn="jit", fixed=False)
    sb = lambda net: sum(t.numel() * t.element_size() for t in net.state.values()
                         if isinstance(t, torch.Tensor))
    assert sb(merged) == sb(plain)
    assert merged.state["g_e"].numel() == n
    # per-projection conductances would need 4 arrays of n fp32 instead of 2;
    # the library's buckets grow by the two extra overflow-count classes only
    slots = 2
    assert merged.device_bytes() <= plain.device_bytes() + slots * 2 * 4 * n + 4096


@pytest.mark.parametrize("delay", [1, 2, 4])
@pytest.mark.parametrize("mode", ["fix64", "f32"])
def test_nccl_exchange_world1_bit_exact(orc, delay, mode):
    """The library-owned NCCL exchange (bp_network_create with
    BP_EXCHANGE_NCCL, world 1: communicator, comm stream, all-gather of the
    own words, the D >= 2 alternating vectors) gives the same network as
    the plain loop and the oracle."""
    n, steps = 20_000, 300
    fixed = {"fix64": True, "f32": False}[mode]
    a = CobaNetwork(n, conn="jit", fixed=fixed, delay=delay, exchange="nccl")
    b = CobaNetwork(n, conn="jit", fixed=fixed, delay=delay)
    ra = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    rb = torch.zeros_like(ra)
    a.run(steps // 2, ra[:steps // 2])
    a.run(steps - steps // 2, ra[steps // 2:])
    b.run(steps, rb)
    assert torch.equal(ra, rb)
    for k in ("v", "g_e", "g_i", "ref"):
        assert torch.equal(a.state[k], b.state[k]), k
    assert a.counters() == b.counters()


@pytest.mark.parametrize("mode", ["fix64", "f32"])
def test_eight_projections_overlapping_and_empty(orc, mode):
    """The most projections a network takes (8), one of them empty, two whose
    presynaptic ranges overlap (rows in both deliver twice), CSR and JIT
    mixed, four weight classes: bit-exact against the oracle's merge."""
    n, steps = 12_000, 250
    p = 80.0 / n
    K = orc.conn_len(p)
    rows = [(0, 3000, "exc", 0.6, "jit"), (3000, 6000, "exc", 0.6, "jit"),
            (6000, 9600, "exc", 0.45, "csr"), (2000, 2500, "exc", 0.45, "jit"),
            (9600, 9600, "exc", 0.6, "jit"),                      # empty
            (9600, 10800, "inh", 6.7, "jit"), (10800, n, "inh", 6.7, "csr"),
            (9000, 11000, "inh", 5.0, "jit")]
    specs, oproj = [], []
    for k, (b, e, rec, w, kind) in enumerate(rows):
        jit = orc.JitSpec(500 + k, K, n, orc.LAW_HOMO, w)
        if kind == "csr":
            ip, ix, _ = orc.jit_materialize(jit, e - b, n)
            specs.append(ProjSpec(b, e, rec, w, csr=(torch.from_numpy(ip), torch.from_numpy(ix))))
            oproj.append(orc.Projection(b, e - b, csr=(ip, ix, None), w_homo=w, receptor=rec))
        else:
            specs.append(ProjSpec(b, e, rec, w, seed=500 + k, p=p))
            oproj.append(orc.Projection(b, e - b, jit=jit, receptor=rec))
    net = CobaNetwork(n, conn="jit", fixed={"fix64": True, "f32": False}[mode],
                      projections=specs)
    assert net.net.describe()["classes"] == 4
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, _g(mode)), g_i=np.zeros(n, _g(mode)),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, oproj, None, steps)
    got = np.stack([inputs.unpack_bits(r, n) for r in raster.cpu().numpy().view(np.uint32)])
    assert want.sum() > 0
    assert np.array_equal(got, want)
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(net.state[k].cpu().numpy().view(np.uint8), st[k].view(np.uint8)), k


def test_merged_fp32_weights_off_the_fixed_grid_are_refused():
    """Rule M1: merging fp32 conductances with several weights needs every
    weight on the 2^-32 grid (the exact integer sum); a weight below it is
    refused with BP_ERR_UNSUPPORTED instead of rounding silently."""
    import paper_2311_05106_b200 as bp
    n = 4000
    p = 80.0 / n
    specs = [ProjSpec(0, 2000, "exc", 0.6, seed=1, p=p),
             ProjSpec(2000, 3200, "exc", 1e-12, seed=2, p=p),
             ProjSpec(3200, n, "inh", 6.7, seed=3, p=p)]
    with pytest.raises(bp.BpError, match="UNSUPPORTED"):
        CobaNetwork(n, conn="jit", fixed=False, projections=specs)
    CobaNetwork(n, conn="jit", fixed=True, projections=specs)      # fixed point: fine


@pytest.mark.parametrize("case", range(12))
def test_random_networks_bit_exact(orc, case):
    """Seeded random network shapes against the oracle: n not a multiple of
    32 or of the tile, 1-4 projections with random row ranges, receptors,
    weights (on the 2^-32 grid), JIT or CSR, delays 1-4, every conductance
    mode, one or two calls of bp_network_step."""
    rng = np.random.default_rng(9000 + case)
    n = int(rng.integers(4097, 30_000))
    mode = ["fix64", "fix32", "f32"][case % 3]
    delay = int(rng.integers(1, 5))
    p = float(rng.uniform(40, 120)) / n
    K = orc.conn_len(p)
    n_proj = int(rng.integers(1, 5))
    specs, oproj = [], []
    for k in range(n_proj):
        b = int(rng.integers(0, n - 100))
        e = int(rng.integers(b + 1, n + 1))
        rec = "exc" if rng.random() < 0.6 else "inh"
        w = float(np.float32(rng.choice([0.25, 0.5, 0.75, 1.0, 2.5, 5.0])))
        jit = orc.JitSpec(1000 * case + k, K, n, orc.LAW_HOMO, w)
        if rng.random() < 0.3:
            ip, ix, _ = orc.jit_materialize(jit, e - b, n)
            specs.append(ProjSpec(b, e, rec, w, csr=(torch.from_numpy(ip), torch.from_numpy(ix))))
            oproj.append(orc.Projection(b, e - b, csr=(ip, ix, None), w_homo=w, receptor=rec))
        else:
            specs.append(ProjSpec(b, e, rec, w, seed=1000 * case + k, p=p))
            oproj.append(orc.Projection(b, e - b, jit=jit, receptor=rec))
    classes = {(s.receptor, s.weight) for s in specs}
    if len(classes) > 4:
        pytest.skip("more than 4 weight classes")
    steps = 200
    net = CobaNetwork(n, conn="jit", fixed={"fix64": True, "fix32": "fix32", "f32": False}[mode],
                      projections=specs, delay=delay)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    cut = int(rng.integers(1, steps))
    net.run(cut, raster[:cut])
    net.run(steps - cut, raster[cut:])
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, _g(mode)), g_i=np.zeros(n, _g(mode)),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, oproj, None, steps, delay=delay)
    got = np.stack([inputs.unpack_bits(r, n) for r in raster.cpu().numpy().view(np.uint32)])
    assert np.array_equal(got, want), (n, mode, delay, n_proj)
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(net.state[k].cpu().numpy().view(np.uint8), st[k].view(np.uint8)), k
