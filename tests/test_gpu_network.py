"""GPU parity of the network step (rule S1: Listing S3's update loop) against
the oracle's run_network.

Fixed-point mode (BP_OUT_FIX64) is the primary parity mode: rasters, V bits
and g are bit-exact for every step.  fp32 mode (fp32 atomics) follows rule
T3: rasters identical over the first 200 steps and the population rate
within 1 % over 1 s (north_star).
"""
import numpy as np
import pytest
import torch

from paper_2311_05106_b200 import inputs
from paper_2311_05106_b200.network import SEED_E, SEED_I, CobaNetwork, partition

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)


def _g_dtype(fixed):
    return {True: np.int64, "fix64": np.int64, "fix32": np.int32, False: np.float32,
            "f32": np.float32}[fixed]


def _oracle_lif(orc, n, fixed, csr=None, p=None, w=(0.6, 6.7)):
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n if p is None else p)
    if csr is None:
        pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, n, orc.LAW_HOMO, w[0]))
        pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, n, orc.LAW_HOMO, w[1]))
    else:
        (ipe, ixe), (ipi, ixi) = csr
        pe = orc.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=0.6)
        pi = orc.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=6.7)
    g = _g_dtype(fixed)
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, g), g_i=np.zeros(n, g),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    return st, pe, pi


def _raster(r, n):
    return np.stack([inputs.unpack_bits(row, n) for row in r.cpu().numpy().view(np.uint32)])


@pytest.mark.parametrize("mode", ["fix64", "fix32"])
@pytest.mark.parametrize("n,steps", [(4000, 2000), (1000, 500), (12_345, 300), (4096, 300)])
def test_coba_lif_jit_fixed_bit_exact(orc, n, steps, mode):
    net = CobaNetwork(n, conn="jit", fixed=mode)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, mode)
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    got = _raster(raster, n)
    assert want.sum() > 0
    assert np.array_equal(got, want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
    assert np.array_equal(net.state["g_e"].cpu().numpy(), st["g_e"])
    assert np.array_equal(net.state["g_i"].cpu().numpy(), st["g_i"])
    assert np.array_equal(net.state["ref"].cpu().numpy(), st["ref"])
    spikes, events, saturated = net.counters()
    assert spikes == int(want.sum())            # local spikes emitted (bp_network_counters)
    assert events > 0


@pytest.mark.parametrize("mode", ["fix64", "fix32"])
@pytest.mark.parametrize("small", [True, False])
def test_coba_lif_csr_fixed_bit_exact(orc, small, mode, monkeypatch):
    """small: single-CTA time loop (k_small_net); else k_step + k_bin per step."""
    if not small:
        monkeypatch.setenv("BP_NO_SMALL_NET", "1")
    n, steps = 4000, 1000
    n_exc = 3200
    ipe, ixe, _ = inputs.random_csr(n_exc, n, 0.02, seed=1)
    ipi, ixi, _ = inputs.random_csr(n - n_exc, n, 0.02, seed=2)
    csr = ((ipe, ixe), (ipi, ixi))
    net = CobaNetwork(n, conn="csr", fixed=mode, csr=csr)
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, mode, csr=csr)
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))


@pytest.mark.parametrize("n,steps", [(4000, 10_000), (20_000, 1000)])
def test_coba_lif_f32_bit_exact(orc, n, steps):
    """fp32 conductances with the rule N1-f32 increment fl32(count * w):
    bit-exact over 1 s (which implies T3: identical rasters for 200 steps
    and the rate within 1 %)."""
    net = CobaNetwork(n, conn="jit", fixed=False)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, False)
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    got = _raster(raster, n)
    assert want.sum() > 0
    assert np.array_equal(got, want)
    assert np.array_equal(net.state["g_e"].cpu().numpy().view(np.uint32), st["g_e"].view(np.uint32))
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))


@pytest.mark.parametrize("path", ["small", "dense", "tiles"])
@pytest.mark.parametrize("fixed", ["fix64", "fix32", "f32"])
def test_coba_hh_csr(orc, fixed, path, monkeypatch):
    """small: single-CTA loop; dense: per-neuron event counts + 512-neuron
    blocks (the HH default beyond one CTA); tiles: 4096-neuron tiles with
    event buckets."""
    if path != "small":
        monkeypatch.setenv("BP_NO_SMALL_NET", "1")
    if path == "tiles":
        monkeypatch.setenv("BP_DENSE", "0")
    n, steps = 4000, 400
    orc.set_fix32_bits(16)
    n_exc = 3200
    ipe, ixe, _ = inputs.random_csr(n_exc, n, 0.02, seed=11)
    ipi, ixi, _ = inputs.random_csr(n - n_exc, n, 0.02, seed=12)
    net = CobaNetwork(n, model="hh", conn="csr", fixed=fixed, csr=((ipe, ixe), (ipi, ixi)))
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    v, m, h, nk = inputs.hh_init(n)
    g = _g_dtype(fixed)
    st = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, g), g_i=np.zeros(n, g),
              spikes=np.zeros(n, np.uint8))
    pe = orc.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=6.0)
    pi = orc.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=67.0)
    want = orc.run_network("hh", orc.hh_params(), st, pe, pi, steps)
    orc.set_fix32_bits(20)
    got = _raster(raster, n)
    assert want.sum() > 0
    assert net.counters()[2] == 0          # no FIX32 saturation
    assert np.array_equal(got, want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))


def test_split_step_equals_fused_step(orc):
    """bp_network_scatter + bp_network_update (the multi-GPU halves, with no
    exchange at world 1) reproduce bp_network_step."""
    n, steps = 3000, 300
    a = CobaNetwork(n, conn="jit", fixed=True)
    b = CobaNetwork(n, conn="jit", fixed=True)
    a.run(steps)
    for _ in range(steps):
        b.net.scatter()
        b.net.update()
    assert np.array_equal(a.state["v"].cpu().numpy(), b.state["v"].cpu().numpy())
    assert np.array_equal(a.state["g_e"].cpu().numpy(), b.state["g_e"].cpu().numpy())


@pytest.mark.parametrize("compact", ["0", "1"])
@pytest.mark.parametrize("n,steps", [(4096, 300), (50_000, 120)])
def test_partitions_emulated_on_one_gpu_equal_whole(orc, monkeypatch, compact, n, steps):
    """G postsynaptic partitions stepped one after another on one device,
    with the all-gather emulated by sharing one spike vector, give the
    single-partition network bit for bit.  The remote
    rows are listed by the binning blocks themselves (BP_BIN_COMPACT=0) or
    compacted by a separate launch (1); n = 50 000 has a ragged last word."""
    monkeypatch.setenv("BP_BIN_COMPACT", compact)
    world = 4
    whole = CobaNetwork(n, conn="jit", fixed=True, seg_len=1024)
    whole.run(steps)
    shared = torch.zeros(partition(n, world, 0, 1024).padded_words, dtype=torch.int32,
                         device="cuda")
    parts = [CobaNetwork(n, conn="jit", fixed=True, seg_len=1024, rank=r, world=world,
                         spikes=shared) for r in range(world)]
    for _ in range(steps):
        for q in parts:          # every rank scatters spikes_{n-1} first ...
            q.net.scatter()
        for q in parts:          # ... then all update (the exchange is the shared vector)
            q.net.update()
    v = np.concatenate([q.state["v"].cpu().numpy() for q in parts])
    assert np.array_equal(v.view(np.uint32), whole.state["v"].cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("group", ["", "2", "4"])
def test_weak_partitions_item_lanes_equal_whole(orc, monkeypatch, group):
    """8 partitions whose segment is the whole partition (the weak-scaling
    layout) with ~10 events per (row, segment): the binning's 2-lanes-per-
    item split (the default for such networks from 16 M neurons) and the
    4-lane one (the default at this size) give the whole network's state
    bit for bit; the whole network checks against the oracle's raster."""
    n, world, steps, L = 80_000, 8, 150, 10_016
    whole = CobaNetwork(n, conn="jit", fixed=True, seg_len=L)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    whole.run(steps, raster)
    if group:
        monkeypatch.setenv("BP_BIN_GROUP", group)
    shared = torch.zeros(partition(n, world, 0, L).padded_words, dtype=torch.int32,
                         device="cuda")
    parts = [CobaNetwork(n, conn="jit", fixed=True, seg_len=L, rank=r, world=world,
                         spikes=shared) for r in range(world)]
    if not group:
        assert parts[0].net.describe()["bin_lanes"] == 4
    for _ in range(steps):
        for q in parts:
            q.net.scatter()
        for q in parts:
            q.net.update()
    v = np.concatenate([q.state["v"].cpu().numpy() for q in parts])[:n]
    assert np.array_equal(v.view(np.uint32), whole.state["v"].cpu().numpy().view(np.uint32))
    ge = np.concatenate([q.state["g_e"].cpu().numpy() for q in parts])[:n]
    assert np.array_equal(ge, whole.state["g_e"].cpu().numpy())
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, L, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, L, orc.LAW_HOMO, 6.7))
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)


@pytest.mark.parametrize("cap", ["1", "8", "64"])
def test_bucket_overflow_spill_is_exact(orc, monkeypatch, cap):
    """Tiles receiving more events than their bucket holds spill into dense
    counters; the result must stay bit-exact (step.cuh)."""
    monkeypatch.setenv("BP_BUCKET_CAP", cap)
    n, steps = 8192, 300
    net = CobaNetwork(n, conn="jit", fixed=True)
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, True)
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["g_i"].cpu().numpy(), st["g_i"])


def test_step_counts_out(orc):
    n, steps = 4000, 200
    net = CobaNetwork(n, conn="jit", fixed=True)
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    counts = torch.zeros(steps, dtype=torch.int32).pin_memory()
    net.run(steps, raster, counts)
    torch.cuda.synchronize()
    got = _raster(raster, n).sum(axis=1)
    assert np.array_equal(counts.numpy(), got)


# ---------------------------------------------------- NEXT 2: synaptic delays
@pytest.mark.parametrize("mode", ["fix64", "f32"])
@pytest.mark.parametrize("delay", [2, 5, 16])
@pytest.mark.parametrize("n,steps", [(4000, 600), (20_000, 300)])
def test_coba_lif_delay_bit_exact(orc, n, steps, delay, mode):
    """Reading D1: spikes of step n arrive at step n + D (D + 1 bucket slots)."""
    net = CobaNetwork(n, conn="jit", fixed={"fix64": True, "f32": False}[mode], delay=delay)
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps // 3, raster[:steps // 3])               # two calls: the ring carries over
    net.run(steps - steps // 3, raster[steps // 3:])
    st, pe, pi = _oracle_lif(orc, n, {"fix64": True, "f32": False}[mode])
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps, delay=delay)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
    assert np.array_equal(net.state["g_e"].cpu().numpy().view(np.uint32 if mode == "f32" else np.int64),
                          st["g_e"].view(np.uint32 if mode == "f32" else np.int64))


def test_delay_partitions_emulated_equal_whole(orc):
    """Delayed network over 4 postsynaptic partitions (exchange emulated by a
    shared spike vector) equals the single partition bit for bit."""
    n, steps, world, delay = 4096, 200, 4, 3
    whole = CobaNetwork(n, conn="jit", fixed=True, seg_len=1024, delay=delay)
    whole.run(steps)
    shared = torch.zeros(n // 32, dtype=torch.int32, device="cuda")
    parts = [CobaNetwork(n, conn="jit", fixed=True, seg_len=1024, rank=r, world=world,
                         spikes=shared, delay=delay) for r in range(world)]
    for _ in range(steps):
        for q in parts:
            q.net.scatter()
        for q in parts:
            q.net.update()
    v = np.concatenate([q.state["v"].cpu().numpy() for q in parts])
    assert np.array_equal(v.view(np.uint32), whole.state["v"].cpu().numpy().view(np.uint32))


@pytest.mark.parametrize("mode", ["fix64", "f32"])
def test_coba_lif_dense_delivery_bit_exact(orc, mode, monkeypatch):
    """Dense delivery forced for the LIF network (ragged last block)."""
    monkeypatch.setenv("BP_DENSE", "1")
    n, steps = 20_001 - 20_001 % 32 + 32, 300
    net = CobaNetwork(n, conn="jit", fixed={"fix64": True, "f32": False}[mode])
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, {"fix64": True, "f32": False}[mode])
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))


# Fig S3B / S3C regimes (NEXT 4): 1000 synapses per neuron, and a
# fixed p = 0.001, weights rescaled by 80 / fan-in (reading R29).
@pytest.mark.parametrize("mode", ["fix64", "f32"])
@pytest.mark.parametrize("n,p,steps", [(20_000, 0.05, 400),      # fan-in 1000 (S3B)
                                       (100_000, 0.001, 200),    # p = 0.001 (S3C)
                                       (50_000, 0.02, 200)])     # fan-in 1000 again, 2 tiles+
def test_fig_s3_regimes_bit_exact(orc, n, p, steps, mode):
    scale = 80.0 / (p * n)
    w = (0.6 * scale, 6.7 * scale)
    net = CobaNetwork(n, conn="jit", fixed=mode, p=p, w_exc=w[0], w_inh=w[1])
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    st, pe, pi = _oracle_lif(orc, n, mode, p=p, w=w)
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    got = _raster(raster, n)
    assert want.sum() > 0
    assert np.array_equal(got, want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
    g = net.state["g_e"].cpu().numpy()
    assert np.array_equal(g.view(np.uint32) if mode == "f32" else g,
                          st["g_e"].view(np.uint32) if mode == "f32" else st["g_e"])


@pytest.mark.parametrize("group", ["", "4", "32", "64"])
def test_segmented_long_items_bit_exact(orc, monkeypatch, group):
    """Rows of several long JIT segments (fan-in 1000, seg_len 4992 -> 5
    segments, the last one 32 columns; ~250 events per (row, segment)):
    every binning work split -- 4 lanes per item, a warp per row walking its
    segments, a warp per (row, segment) item (the default here) -- gives the
    oracle's raster and state bit for bit."""
    if group:
        monkeypatch.setenv("BP_BIN_GROUP", group)
    n, p, steps, L = 20_000, 0.05, 300, 4992
    scale = 80.0 / (p * n)
    w = (0.6 * scale, 6.7 * scale)
    net = CobaNetwork(n, conn="jit", fixed=True, p=p, w_exc=w[0], w_inh=w[1], seg_len=L)
    if not group:
        assert net.net.describe()["bin_lanes"] == 64
    raster = torch.zeros((steps, (n + 31) // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    n_exc = n * 4 // 5
    K = orc.conn_len(p)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, L, orc.LAW_HOMO, w[0]))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(SEED_I, K, L, orc.LAW_HOMO, w[1]))
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, steps)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["g_e"].cpu().numpy(), st["g_e"])


def test_execution_plan_choices():
    """bp_network_describe: the single-CTA loop for <= 4096 neurons, dense
    delivery for HH up to 2 M local neurons and tiles beyond (the
    dense-before-n_local ordering bug of round 1 forced dense for every HH
    network), 4 lanes per binning item for few events per segment."""
    small = CobaNetwork(4000, conn="jit", fixed=True).net.describe()
    assert small["small"] == 1
    lif = CobaNetwork(50_000, conn="jit", fixed=False).net.describe()
    assert lif["small"] == 0 and lif["dense"] == 0 and lif["n_tiles"] == 13
    assert lif["bin_lanes"] == 32 and lif["fold_classes"] == 2
    hh = CobaNetwork(100_000, model="hh", conn="jit", fixed=False).net.describe()
    assert hh["dense"] == 1
    big = CobaNetwork((2 << 20) + 64, model="hh", conn="jit", fixed=False, seg_len=None)
    assert big.net.describe()["dense"] == 0
    seg8 = CobaNetwork(400_000, conn="jit", fixed=False, seg_len=50_000).net.describe()
    assert seg8["bin_lanes"] == 4


def test_remote_listing_burst_matches_compaction(monkeypatch):
    """Every neuron of a 4 M network spikes at once: rank 0 of 4 bins ~3 M
    remote rows, ~20 k per binning block -- more than one listing round of
    the block's shared list and more events than its staging area (the
    per-event overflow, and the buckets' dense spill).  The in-kernel
    listing and the compaction launch must give the same conductances and
    event count bit for bit."""
    n, world = 4_000_000, 4
    got = []
    for compact in ("0", "1"):
        monkeypatch.setenv("BP_BIN_COMPACT", compact)
        shared = torch.full(((n + 31) // 32,), -1, dtype=torch.int32, device="cuda")
        q = CobaNetwork(n, conn="jit", fixed=True, seg_len=n // world, rank=0, world=world,
                        spikes=shared)
        q.net.scatter()
        q.net.update()
        torch.cuda.synchronize()
        _, events, _ = q.counters()
        got.append((q.state["g_e"].cpu().numpy(), q.state["g_i"].cpu().numpy(), events))
        del q, shared
    (ge0, gi0, ev0), (ge1, gi1, ev1) = got
    assert ev0 == ev1 and ev0 > (3 * n // 4) * 15   # ~20 local events per remote row
    assert np.array_equal(ge0, ge1) and np.array_equal(gi0, gi1)
    assert ge0.any()


@pytest.mark.parametrize("compact", ["0", "1"])
def test_hh_partitions_emulated_equal_oracle(orc, monkeypatch, compact):
    """HH network (dense delivery) over 4 postsynaptic partitions with the
    exchange emulated by a shared spike vector: the remote rows go through
    the per-event word-listing kernel (BP_BIN_COMPACT=0) or compaction +
    per-row binning (1); the raster equals the oracle's bit for bit."""
    monkeypatch.setenv("BP_BIN_COMPACT", compact)
    n, steps, world = 4000, 300, 4
    n_exc = 3200
    ipe, ixe, _ = inputs.random_csr(n_exc, n, 0.02, seed=11)
    ipi, ixi, _ = inputs.random_csr(n - n_exc, n, 0.02, seed=12)
    shared = torch.zeros(partition(n, world, 0).padded_words, dtype=torch.int32, device="cuda")
    parts = [CobaNetwork(n, model="hh", conn="csr", fixed=True, csr=((ipe, ixe), (ipi, ixi)),
                         rank=r, world=world, spikes=shared) for r in range(world)]
    raster = np.zeros((steps, n), np.uint8)
    for t in range(steps):
        for q in parts:
            q.net.scatter()
        for q in parts:
            q.net.update()
        torch.cuda.synchronize()
        raster[t] = inputs.unpack_bits(shared.cpu().numpy().view(np.uint32)[:(n + 31) // 32], n)
    v, m, h, nk = inputs.hh_init(n)
    st = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
              spikes=np.zeros(n, np.uint8))
    pe = orc.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=6.0)
    pi = orc.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=67.0)
    want = orc.run_network("hh", orc.hh_params(), st, pe, pi, steps)
    assert want.sum() > 0
    assert np.array_equal(raster, want)
    v_got = np.concatenate([q.state["v"].cpu().numpy() for q in parts])
    assert np.array_equal(v_got.view(np.uint32), st["v"].view(np.uint32))


@pytest.mark.parametrize("fused", ["1", "0"])
@pytest.mark.parametrize("delay", [1, 3])
def test_hh_dense_delivery_with_delay_bit_exact(orc, monkeypatch, fused, delay):
    """Dense HH delivery (the update kernel delivering its own spikes, or the
    separate binning launch) into the bucket ring of reading D1: spikes of
    step n arrive at step n + D; raster and V equal the oracle's."""
    monkeypatch.setenv("BP_NO_SMALL_NET", "1")
    monkeypatch.setenv("BP_HH_FUSED", fused)
    n, steps = 4000, 300
    n_exc = 3200
    ipe, ixe, _ = inputs.random_csr(n_exc, n, 0.02, seed=11)
    ipi, ixi, _ = inputs.random_csr(n - n_exc, n, 0.02, seed=12)
    net = CobaNetwork(n, model="hh", conn="csr", fixed=True, csr=((ipe, ixe), (ipi, ixi)),
                      delay=delay)
    assert net.net.describe()["dense"] == 1
    raster = torch.zeros((steps, n // 32), dtype=torch.int32, device="cuda")
    net.run(steps, raster)
    v, m, h, nk = inputs.hh_init(n)
    st = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
              spikes=np.zeros(n, np.uint8))
    pe = orc.Projection(0, n_exc, csr=(ipe, ixe, None), w_homo=6.0)
    pi = orc.Projection(n_exc, n - n_exc, csr=(ipi, ixi, None), w_homo=67.0)
    want = orc.run_network("hh", orc.hh_params(), st, pe, pi, steps, delay=delay)
    assert want.sum() > 0
    assert np.array_equal(_raster(raster, n), want)
    assert np.array_equal(net.state["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
