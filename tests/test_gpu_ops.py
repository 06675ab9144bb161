"""GPU parity of the stateless C-ABI operators against the CPU oracle.

Bars: index sets, positions and every BP_OUT_FIX64
output are bit-exact; BP_OUT_F32 outputs satisfy rule T2,
|y_gpu - y_f64| <= 1e-5 * sum|w| + 1e-30 per output (order-free bound for
fp32 atomics).  Weights of every law (normal: the fp32 Box-Muller of
reading J7n) are bit-identical on both sides.
"""
import numpy as np
import pytest
import torch

from paper_2311_05106_b200 import inputs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def bp():
    import __graft_entry__ as ge
    ge.build_lib()
    import paper_2311_05106_b200 as bp
    torch.cuda.set_device(0)
    return bp


def _dev_spikes(ev):
    return torch.from_numpy(inputs.pack_bits(ev).view(np.int32)).cuda()


def _t(a):
    return None if a is None else torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ------------------------------------------------------------------ a1
@pytest.mark.parametrize("n", [1, 31, 32, 33, 1000, 100_003, 3_000_017])
@pytest.mark.parametrize("density", [0.0, 0.001, 0.3, 1.0])
def test_compact_is_the_active_set(bp, n, density):
    ev = inputs.spike_pattern(n, density, seed=n)
    spikes = _dev_spikes(ev)
    active = torch.full((n,), -1, dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")
    bp.compact_spikes(spikes, n, active, count)
    c = int(count.item())
    got = np.sort(active[:c].cpu().numpy())
    assert np.array_equal(got, np.nonzero(ev)[0].astype(np.int32))


def test_compact_ignores_tail_bits(bp):
    words = torch.full((2,), -1, dtype=torch.int32, device="cuda")   # 64 set bits
    active = torch.zeros(40, dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")
    bp.compact_spikes(words, 40, active, count)
    assert int(count.item()) == 40


# ------------------------------------------------------------------ a2
CSR_CASES = [
    # n_rows, n_cols, p, weights, density
    (1, 1, 1.0, "homo", 1.0),
    (50, 70, 0.2, "homo", 0.5),
    (300, 5000, 0.05, "uniform", 0.1),    # rows of ~250: several 128-wide chunks + tail
    (2000, 3000, 0.01, "normal", 0.01),
    (4000, 4000, 0.02, "homo", 0.002),
    (1000, 100_000, 0.05, "uniform", 0.05),   # fan-out 5000 (config 2 row shape)
    (300, 500_000, 0.01, "uniform", 0.3),     # many column tiles
    (500, 2_000_000, 0.001, "homo", 0.2),     # > 16 tiles: direct path
    (20_000, 1000, 0.01, "uniform", 1.0),     # short rows: 16-piece stages
    (64, 33_333, 0.5, "homo", 1.0),           # rows of ~16k: pieces span stages
]


@pytest.mark.parametrize("path", ["stream", "planned", "stream_nofuse", "tiled", "atomic_flush",
                                  "direct", "unaligned"])
@pytest.mark.parametrize("case", CSR_CASES)
def test_event_csrmv(bp, orc, case, path, monkeypatch):
    """stream: bulk-copy streamed column tiles + ordered partial reduction
    (default, partials reduced inside the cooperative kernel); planned: the
    same with split points precomputed by csrmv_plan; stream_nofuse:
    the same with a separate reduction kernel; tiled: register-staged tiles
    + reduction; atomic_flush: tiles
    flushed with REDs; direct: one RED per event; unaligned: indices/data not
    16-byte aligned (the bulk-copy path must step aside)."""
    if path == "direct":
        monkeypatch.setenv("BP_CSR_DIRECT", "1")
    if path == "atomic_flush":
        monkeypatch.setenv("BP_CSR_ATOMIC_FLUSH", "1")
    if path == "tiled":
        monkeypatch.setenv("BP_CSR_TILED", "1")
    if path == "stream_nofuse":
        monkeypatch.setenv("BP_CSR_NO_FUSE", "1")
    n_rows, n_cols, p, law, density = case
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, p, seed=n_rows + n_cols,
                                    weights=law, w0=-0.5 if law != "homo" else 1.0,
                                    w1=0.5 if law != "homo" else 0.0)
    w_homo = 0.6
    ev = inputs.spike_pattern(n_rows, density, seed=3)
    spikes = _dev_spikes(ev)
    tip, tix, tdat = _t(ip), _t(ix), _t(dat)
    if path == "unaligned":          # same values, views offset by one element
        tix = torch.cat([tix.new_zeros(1), tix])[1:]
        tdat = None if tdat is None else torch.cat([tdat.new_zeros(1), tdat])[1:]
    plan64 = plan32 = None
    if path == "planned":
        plan64 = bp.csrmv_plan(tip, tix, n_rows, n_cols, torch.int64, homo=tdat is None, data=tdat)
        plan32 = bp.csrmv_plan(tip, tix, n_rows, n_cols, torch.float32, homo=tdat is None, data=tdat)
    # fixed point: bit-exact
    out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    bp.event_csrmv(tip, tix, tdat, w_homo, n_rows, n_cols, spikes, out, plan=plan64)
    want = orc.event_csrmv(ip, ix, dat, w_homo, n_rows, n_cols, ev, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want)
    # fp32 atomics: rule T2
    out32 = torch.full((n_cols,), 7.0, dtype=torch.float32, device="cuda")
    bp.event_csrmv(tip, tix, tdat, w_homo, n_rows, n_cols, spikes, out32, plan=plan32)
    ref, absw = orc.event_csrmv(ip, ix, dat, w_homo, n_rows, n_cols, ev, orc.OUT_F64,
                                with_abs=True)
    err = np.abs(out32.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)


def test_event_csrmv_accumulate_and_empty(bp, orc):
    ip, ix, _ = inputs.random_csr(100, 64, 0.3, seed=1)
    ev = inputs.spike_pattern(100, 0.2, 2)
    out = torch.full((64,), 5 * 2 ** 32, dtype=torch.int64, device="cuda")
    bp.event_csrmv(_t(ip), _t(ix), None, 1.5, 100, 64, _dev_spikes(ev), out, accumulate=True)
    want = orc.event_csrmv(ip, ix, None, 1.5, 100, 64, ev, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want + 5 * 2 ** 32)
    # all-false events and n_rows = 0 leave a zeroed output
    out.fill_(123)
    bp.event_csrmv(_t(ip), _t(ix), None, 1.5, 100, 64,
                   _dev_spikes(np.zeros(100, np.uint8)), out)
    assert not out.any()
    out.fill_(123)
    bp.event_csrmv(_t(np.zeros(1, np.int64)), _t(np.zeros(1, np.int32)), None, 1.0,
                   0, 64, _dev_spikes(np.zeros(1, np.uint8)), out)
    assert not out.any()


def test_event_csrmv_rejects_bad_arguments(bp):
    out = torch.zeros(8, dtype=torch.float64, device="cuda")
    with pytest.raises(bp.BpError):
        bp.event_csrmv(_t(np.zeros(2, np.int64)), _t(np.zeros(1, np.int32)), None,
                       1.0, 1, 8, _dev_spikes(np.ones(1, np.uint8)), out)
    with pytest.raises(bp.BpError, match="WORKSPACE"):
        bp.event_csrmv(_t(np.zeros(2, np.int64)), _t(np.zeros(1, np.int32)), None,
                       1.0, 1, 8, _dev_spikes(np.ones(1, np.uint8)),
                       torch.zeros(8, device="cuda"),
                       ws=torch.zeros(16, dtype=torch.uint8, device="cuda"))


# ------------------------------------------------------------------ a3 + a4
JIT_CASES = [
    # n_rows, n_cols, p, seg_len, density
    (64, 37, 1.0, 0, 0.5),             # K = 1: dense rows
    (500, 3000, 0.05, 0, 0.1),         # fan-out 150 > 128: two chunks
    (300, 10_000, 0.1, 1000, 0.2),     # 10 segments
    (1000, 100_000, 0.05, 0, 0.01),    # fan-out 5000 (config 2 row shape)
    (4000, 4000, 0.02, 0, 0.01),       # COBA-4000 projection shape
    (3, 2**20, 80 / 2**20, 0, 1.0),    # huge K = 26213; > 16 column tiles: per-event path
    (200, 300_000, 0.005, 0, 0.1),     # 6-11 column tiles, rows spanning all of them
    (150, 240_000, 0.01, 40_000, 0.2), # segments shorter than a tile
]


@pytest.mark.parametrize("path", ["tiled", "direct"])
@pytest.mark.parametrize("case", JIT_CASES)
@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
def test_jitconn_event_mv(bp, orc, case, law, path, monkeypatch):
    """tiled: shared-memory column tiles + in-kernel reduction (default when
    the workspace holds the partial tiles); direct: one global RED per event."""
    if path == "direct":
        monkeypatch.setenv("BP_JIT_DIRECT", "1")
    else:
        monkeypatch.setenv("BP_JIT_TILED", "1")     # normal weights too
    n_rows, n_cols, p, seg_len, density = case
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-0.1, 0.1), "normal": (0.0, 0.3)}[law]
    seed = 0xC0FFEE + n_rows
    K = orc.conn_len(p)
    L = seg_len or n_cols
    ospec = orc.JitSpec(seed, K, L, orc.LAWS[law], w0, w1)
    spec = bp.jitconn_spec(seed, p, 0, seg_len)
    ev = inputs.spike_pattern(n_rows, density, seed=9)
    spikes = _dev_spikes(ev)
    fn = {"homo": lambda o: bp.jitconn_event_mv_homo(spec, w0, spikes, n_rows, n_cols, o),
          "uniform": lambda o: bp.jitconn_event_mv_uniform(spec, w0, w1, spikes, n_rows, n_cols, o),
          "normal": lambda o: bp.jitconn_event_mv_normal(spec, w0, w1, spikes, n_rows, n_cols, o)}[law]
    out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    fn(out)
    want = orc.jit_event_mv(ospec, n_rows, n_cols, ev, out_kind=orc.OUT_FIX)
    got = out.cpu().numpy()
    assert np.array_equal(got, want)              # every law bit-exact (J7n)
    out32 = torch.zeros(n_cols, dtype=torch.float32, device="cuda")
    fn(out32)
    ref, absw = orc.jit_event_mv(ospec, n_rows, n_cols, ev, out_kind=orc.OUT_F64,
                                 with_abs=True)
    err = np.abs(out32.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)


@pytest.mark.parametrize("path", ["tiled", "direct"])
@pytest.mark.parametrize("bounds", [(0, 1000), (1000, 5000), (9000, 10_000), (2000, 2000)])
def test_jitconn_partition(bp, orc, bounds, path, monkeypatch):
    if path == "direct":
        monkeypatch.setenv("BP_JIT_DIRECT", "1")
    n_rows, n_cols, L = 400, 10_000, 1000
    cb, ce = bounds
    spec = bp.jitconn_spec(77, 0.02, 0, L)
    ospec = orc.JitSpec(77, orc.conn_len(0.02), L, orc.LAW_UNIFORM, -1.0, 1.0)
    ev = inputs.spike_pattern(n_rows, 0.3, seed=4)
    out = torch.zeros(ce - cb, dtype=torch.int64, device="cuda")
    bp.jitconn_event_mv_uniform(spec, -1.0, 1.0, _dev_spikes(ev), n_rows, n_cols, out,
                                col_begin=cb, col_end=ce)
    want = orc.jit_event_mv(ospec, n_rows, n_cols, ev, cb, ce, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("law", ["homo", "uniform"])
def test_jitconn_tiled_accumulate_and_wide_partition(bp, orc, law):
    """Tiled path: accumulate into a non-zero output; a partition of 130 k
    columns (3 tiles) out of 260 k."""
    n_rows, n_cols, L = 300, 260_000, 130_000
    cb, ce = 130_000, 260_000
    w0, w1 = (0.6, 0.0) if law == "homo" else (-0.2, 0.3)
    spec = bp.jitconn_spec(4242, 0.004, 0, L)
    ospec = orc.JitSpec(4242, orc.conn_len(0.004), L, orc.LAWS[law], w0, w1)
    ev = inputs.spike_pattern(n_rows, 0.25, seed=12)
    out = torch.full((ce - cb,), 3 * 2 ** 32, dtype=torch.int64, device="cuda")
    fn = bp.jitconn_event_mv_homo if law == "homo" else bp.jitconn_event_mv_uniform
    args = (spec, w0) if law == "homo" else (spec, w0, w1)
    fn(*args, _dev_spikes(ev), n_rows, n_cols, out, col_begin=cb, col_end=ce, accumulate=True)
    want = orc.jit_event_mv(ospec, n_rows, n_cols, ev, cb, ce, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want + 3 * 2 ** 32)


def test_jitconn_rejects_unaligned_partition(bp):
    spec = bp.jitconn_spec(1, 0.1, 0, 100)
    out = torch.zeros(50, dtype=torch.float32, device="cuda")
    with pytest.raises(bp.BpError, match="SHAPE"):
        bp.jitconn_event_mv_homo(spec, 1.0, _dev_spikes(np.ones(10, np.uint8)), 10, 1000,
                                 out, col_begin=50, col_end=100)
    with pytest.raises(bp.BpError, match="INVALID"):
        bp.jitconn_event_mv_homo(bp.jitconn_spec(1, 1.5), 1.0,
                                 _dev_spikes(np.ones(10, np.uint8)), 10, 1000,
                                 torch.zeros(1000, device="cuda"))


@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
@pytest.mark.parametrize("shape", [(200, 5000, 0.05, 0), (100, 4000, 0.1, 300), (50, 37, 1.0, 0)])
def test_materialize_positions_bit_exact(bp, orc, law, shape):
    """The kernel's generator yields exactly the oracle's positions (J4-J6)."""
    n_rows, n_cols, p, seg_len = shape
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-1.0, 1.0), "normal": (0.5, 2.0)}[law]
    L = seg_len or n_cols
    seed = 4242
    ip, ix, dat = bp.jitconn_materialize(bp.jitconn_spec(seed, p, 0, seg_len), n_rows,
                                         n_cols, law=orc.LAWS[law], w0=w0, w1=w1)
    ip, ix, dat = ip.cpu().numpy(), ix.cpu().numpy(), dat.cpu().numpy()
    ospec = orc.JitSpec(seed, orc.conn_len(p), L, orc.LAWS[law], w0, w1)
    oip, oix, odat = orc.jit_materialize(ospec, n_rows, n_cols)
    assert np.array_equal(ip, oip)
    assert np.array_equal(ix, oix)
    assert np.array_equal(dat.view(np.uint32), odat.view(np.uint32))   # J7n: every law


# ------------------------------------------------------------------ a5 + a6
def _rand_lif_state(n, fixed, seed):
    rng = np.random.default_rng(seed)
    v = rng.uniform(-70, -45, n).astype(np.float32)
    if fixed == "fix32":
        ge = rng.integers(0, 5 * 2 ** 20, n).astype(np.int32)
        gi = rng.integers(0, 40 * 2 ** 20, n).astype(np.int32)
    elif fixed:
        ge = rng.integers(0, 5 * 2 ** 32, n).astype(np.int64)
        gi = rng.integers(0, 40 * 2 ** 32, n).astype(np.int64)
    else:
        ge = rng.uniform(0, 5, n).astype(np.float32)
        gi = rng.uniform(0, 40, n).astype(np.float32)
    ref = rng.integers(0, 51, n).astype(np.uint8)
    ref[rng.random(n) < 0.6] = 0
    return dict(v=v, g_e=ge, g_i=gi, ref=ref)


@pytest.mark.parametrize("n", [1, 33, 4000, 100_003])
@pytest.mark.parametrize("fixed", [True, False, "fix32"])
def test_lif_step_bit_exact(bp, orc, n, fixed):
    st = _rand_lif_state(n, fixed, seed=n)
    dev = {k: _t(a) for k, a in st.items()}
    if fixed == "fix32":
        dev["frac_bits"] = 20
        orc.set_fix32_bits(20)
    spikes = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    active = torch.zeros(n, dtype=torch.int32, device="cuda")
    count = torch.zeros(1, dtype=torch.int32, device="cuda")
    params = bp.lif_params()
    bp.neuron_step(params, dev, spikes, active, count, active_base=1000)
    ev = orc.lif_step(orc.lif_params(), st["v"], st["g_e"], st["g_i"], st["ref"])
    assert np.array_equal(dev["v"].cpu().numpy().view(np.uint32), st["v"].view(np.uint32))
    assert np.array_equal(dev["ref"].cpu().numpy(), st["ref"])
    assert np.array_equal(dev["g_e"].cpu().numpy(), st["g_e"])
    assert np.array_equal(dev["g_i"].cpu().numpy(), st["g_i"])
    got = inputs.unpack_bits(spikes.cpu().numpy().view(np.uint32), n)
    assert np.array_equal(got, ev)
    c = int(count.item())
    assert np.array_equal(np.sort(active[:c].cpu().numpy()), np.nonzero(ev)[0] + 1000)


@pytest.mark.parametrize("n", [1, 1000, 65_537])
@pytest.mark.parametrize("fixed", [True, False])
def test_hh_step_bit_exact(bp, orc, n, fixed):
    rng = np.random.default_rng(n)
    v = rng.uniform(-80, 40, n).astype(np.float32)
    v[:3] = np.float32([-50.0, -48.0, -23.0])[: min(3, n)]     # rate singularities
    m = rng.uniform(0, 1, n).astype(np.float32)
    h = rng.uniform(0, 1, n).astype(np.float32)
    nk = rng.uniform(0, 1, n).astype(np.float32)
    if fixed:
        ge = rng.integers(0, 50 * 2 ** 32, n).astype(np.int64)
        gi = rng.integers(0, 300 * 2 ** 32, n).astype(np.int64)
    else:
        ge = rng.uniform(0, 50, n).astype(np.float32)
        gi = rng.uniform(0, 300, n).astype(np.float32)
    st = dict(v=v, m=m, h=h, n=nk, g_e=ge, g_i=gi)
    dev = {k: _t(a) for k, a in st.items()}
    spikes = torch.zeros((n + 31) // 32, dtype=torch.int32, device="cuda")
    for _ in range(3):
        bp.neuron_step(bp.hh_params(), dev, spikes)
        ev = orc.hh_step(orc.hh_params(), st["v"], st["m"], st["h"], st["n"], st["g_e"], st["g_i"])
        for k in ("v", "m", "h", "n"):
            assert np.array_equal(dev[k].cpu().numpy().view(np.uint32), st[k].view(np.uint32)), k
        assert np.array_equal(inputs.unpack_bits(spikes.cpu().numpy().view(np.uint32), n), ev)


# ------------------------------------------------------ NEXT 1: non-event mv
MV_CASES = [
    # n_rows, n_cols, p, seg_len
    (500, 3000, 0.05, 0),
    (300, 100_000, 0.05, 0),          # config-2 row shape, 2 column tiles
    (200, 300_000, 0.005, 0),         # many tiles, rows spanning them
    (150, 240_000, 0.01, 40_000),     # segments shorter than a tile
    (64, 37, 1.0, 0),                 # K = 1: dense
]


@pytest.mark.parametrize("path", ["tiled", "direct"])
@pytest.mark.parametrize("case", MV_CASES)
@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
def test_jitconn_mv(bp, orc, case, law, path, monkeypatch):
    """mv_prob_* (reading MV1) against the oracle: fixed point bit-exact
    (every law), fp32 within rule T2."""
    monkeypatch.setenv("BP_JIT_DIRECT" if path == "direct" else "BP_JIT_TILED", "1")
    n_rows, n_cols, p, seg_len = case
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-0.1, 0.2), "normal": (0.0, 0.3)}[law]
    seed = 0xABC + n_rows
    L = seg_len or n_cols
    ospec = orc.JitSpec(seed, orc.conn_len(p), L, orc.LAWS[law], w0, w1)
    spec = bp.jitconn_spec(seed, p, 0, seg_len)
    rng = np.random.default_rng(n_rows)
    v = rng.normal(0.0, 2.0, n_rows).astype(np.float32)
    v[rng.random(n_rows) < 0.3] = 0.0                 # skipped rows
    tv = _t(v)
    out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    code = {"homo": bp.LAW_HOMO, "uniform": bp.LAW_UNIFORM, "normal": bp.LAW_NORMAL}[law]
    bp.jitconn_mv(code, spec, w0, w1, tv, n_rows, n_cols, out)
    want = orc.jit_mv(ospec, n_rows, n_cols, v, out_kind=orc.OUT_FIX)
    got = out.cpu().numpy()
    assert np.array_equal(got, want)              # every law bit-exact (J7n)
    out32 = torch.zeros(n_cols, dtype=torch.float32, device="cuda")
    bp.jitconn_mv(code, spec, w0, w1, tv, n_rows, n_cols, out32)
    ref, absw = orc.jit_mv(ospec, n_rows, n_cols, v, out_kind=orc.OUT_F64, with_abs=True)
    err = np.abs(out32.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)


def test_jitconn_mv_binary_vector_equals_event_mv(bp):
    """v in {0, 1}: the non-event product is the event scatter, bit for bit."""
    n_rows, n_cols = 400, 100_000
    spec = bp.jitconn_spec(99, 0.05)
    ev = inputs.spike_pattern(n_rows, 0.2, seed=3)
    a = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    b = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    bp.jitconn_event_mv_uniform(spec, -0.3, 0.3, _dev_spikes(ev), n_rows, n_cols, a)
    bp.jitconn_mv(bp.LAW_UNIFORM, spec, -0.3, 0.3, _t(ev.astype(np.float32)), n_rows, n_cols, b)
    assert torch.equal(a, b)


# ------------------------------------------ NEXT 3: gather orientation + grad
GATHER_CASES = [
    # n_rows (outputs), n_cols (event vector), p, weights, density
    (1, 1, 1.0, "homo", 1.0),
    (300, 5000, 0.05, "uniform", 0.1),
    (2000, 3000, 0.01, "homo", 0.3),
    (500, 100_000, 0.02, "uniform", 0.05),
    (10_000, 64, 0.5, "normal", 0.5),        # short rows
]


@pytest.mark.parametrize("case", GATHER_CASES)
def test_csrmv_gather(bp, orc, case):
    n_rows, n_cols, p, law, density = case
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, p, seed=n_rows + 7 * n_cols,
                                    weights=law, w0=-0.5 if law != "homo" else 1.0,
                                    w1=0.5 if law != "homo" else 0.0)
    w = 0.6
    ev = inputs.spike_pattern(n_cols, density, seed=5)
    spikes = _dev_spikes(ev)
    tip, tix, tdat = _t(ip), _t(ix), _t(dat)
    out = torch.full((n_rows,), 3, dtype=torch.int64, device="cuda")
    bp.csrmv_gather(tip, tix, tdat, w, n_rows, n_cols, spikes, out, accumulate=True)
    want = orc.csrmv_gather(ip, ix, dat, w, n_rows, n_cols, ev, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want + 3)
    out32 = torch.zeros(n_rows, dtype=torch.float32, device="cuda")
    bp.csrmv_gather(tip, tix, tdat, w, n_rows, n_cols, spikes, out32)
    ref, absw = orc.csrmv_gather(ip, ix, dat, w, n_rows, n_cols, ev, orc.OUT_F64, with_abs=True)
    assert np.all(np.abs(out32.cpu().numpy() - ref) <= 1e-5 * absw + 1e-30)


@pytest.mark.parametrize("homo", [True, False])
def test_event_csrmv_grad(bp, orc, homo):
    n_rows, n_cols = 3000, 20_000
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.01, seed=31,
                                    weights="homo" if homo else "uniform", w0=-1.0, w1=1.0)
    data = None if homo else dat
    w = 0.6
    ev = inputs.spike_pattern(n_rows, 0.2, seed=6)
    rng = np.random.default_rng(3)
    gy = rng.normal(size=n_cols).astype(np.float32)
    gd = torch.full((ix.shape[0],), 9.0, device="cuda")
    ge = torch.zeros(n_rows, device="cuda")
    gw = torch.full((1,), 5.0, dtype=torch.float64, device="cuda") if homo else None
    bp.event_csrmv_grad(_t(ip), _t(ix), _t(data), w, n_rows, n_cols, _dev_spikes(ev), _t(gy),
                        gd, ge, gw)
    want_gd, want_ge, want_gw = orc.csrmv_grad(ip, ix, data, w, n_rows, ev, gy)
    assert np.array_equal(gd.cpu().numpy(), want_gd)            # exact
    absg = np.zeros(n_rows)
    np.add.at(absg, np.repeat(np.arange(n_rows), np.diff(ip)),
              np.abs((np.float32(w) if homo else dat).astype(np.float64) * gy[ix]))
    assert np.all(np.abs(ge.cpu().numpy() - want_ge) <= 1e-5 * absg + 1e-30)
    if homo:
        tot = np.abs(gy[ix][np.repeat(ev, np.diff(ip)).astype(bool)]).sum()
        assert abs(gw.item() - want_gw) <= 1e-12 * tot + 1e-12


@pytest.mark.parametrize("n_rows", [70_000, 10_000_000])
def test_jitconn_homo_counts_16_bit_boundary(bp, n_rows, monkeypatch):
    """Homogeneous tiles count events in 16 bits while no CTA can reach 2^16
    in one column (k_jit_tiled C16) and fall back to 32 bits beyond (10 M
    dense rows: ~68 k rows per CTA).  Dense rows (p = 1): every column gets
    exactly n_active events, so out = n_active * q(w) in fixed point."""
    monkeypatch.setenv("BP_JIT_TILED", "1")
    n_cols = 40
    spec = bp.jitconn_spec(5, 1.0)
    ev = np.ones(n_rows, np.uint8)
    out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    bp.jitconn_event_mv_homo(spec, 0.25, _dev_spikes(ev), n_rows, n_cols, out)
    assert torch.all(out == n_rows * (2 ** 30)).item()      # q(0.25) = 2^30
    out32 = torch.zeros(n_cols, dtype=torch.float32, device="cuda")
    bp.jitconn_event_mv_homo(spec, 0.25, _dev_spikes(ev), n_rows, n_cols, out32)
    assert torch.all(out32 == np.float32(np.float32(n_rows) * np.float32(0.25))).item()


@pytest.mark.parametrize("c16", [0, 1])
@pytest.mark.parametrize("n_rows", [100_000, 12_000_000])
def test_event_csrmv_homo_counts_16_bit_boundary(bp, n_rows, c16, monkeypatch):
    """The streamed CSR tiles count homogeneous events in 16 bits while a CTA
    streams < 2^16 rows (k_csr_stream C16), 32 bits beyond (12 M dense rows
    of 40 columns).  out = n_active * q(w) exactly.  16-bit counts are
    opt-in (BP_CSR_C16=1); both modes are tested."""
    monkeypatch.setenv("BP_CSR_C16", str(c16))
    n_cols = 40
    indptr = torch.arange(0, n_cols * (n_rows + 1), n_cols, dtype=torch.int64, device="cuda")
    indices = torch.arange(n_cols, dtype=torch.int32, device="cuda").repeat(n_rows)
    ev = np.ones(n_rows, np.uint8)
    for plan in (False, True):
        pl = bp.csrmv_plan(indptr, indices, n_rows, n_cols, torch.int64, homo=True) if plan else None
        out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
        bp.event_csrmv(indptr, indices, None, 0.25, n_rows, n_cols, _dev_spikes(ev), out, plan=pl)
        assert torch.all(out == n_rows * (2 ** 30)).item()
    del indices
    torch.cuda.empty_cache()


@pytest.mark.parametrize("scale", [1.0, 1e-4, 1e4])
def test_csrmv_plan_t4_fixed_point_fp32(bp, orc, scale):
    """Rule T4: a planned heterogeneous fp32 event_csrmv accumulates
    rint(w 2^F) exactly in two 32-bit words per column (F from the plan's
    column bound) and rounds once: within rule T2 of the fp64 definition,
    bitwise identical from call to call (order-free), and ACCUMULATE adds."""
    n_rows, n_cols = 3000, 50_000
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.05, seed=11, weights="uniform",
                                    w0=-scale, w1=scale)
    tip, tix, tdat = _t(ip), _t(ix), _t(dat)
    plan = bp.csrmv_plan(tip, tix, n_rows, n_cols, torch.float32, homo=False, data=tdat)
    assert plan is not None and plan.f32_fixed_bits >= 8
    assert plan.info.max_col_abs_sum > 0
    ev = inputs.spike_pattern(n_rows, 0.3, 4)
    spikes = _dev_spikes(ev)
    a = torch.zeros(n_cols, dtype=torch.float32, device="cuda")
    b = torch.zeros_like(a)
    bp.event_csrmv(tip, tix, tdat, 0.0, n_rows, n_cols, spikes, a, plan=plan)
    bp.event_csrmv(tip, tix, tdat, 0.0, n_rows, n_cols, spikes, b, plan=plan)
    assert torch.equal(a.view(torch.int32), b.view(torch.int32))
    ref, absw = orc.event_csrmv(ip, ix, dat, 0.0, n_rows, n_cols, ev, orc.OUT_F64, with_abs=True)
    err = np.abs(a.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)
    c = torch.full((n_cols,), 7.0 * scale, dtype=torch.float32, device="cuda")
    bp.event_csrmv(tip, tix, tdat, 0.0, n_rows, n_cols, spikes, c, plan=plan, accumulate=True)
    err = np.abs(c.cpu().numpy().astype(np.float64) - (ref + np.float32(7.0 * scale)))
    assert np.all(err <= 1e-5 * (absw + 7.0 * scale))


def test_csrmv_plan_t4_falls_back_for_unbounded_sums(bp, orc):
    """Column sums too large for the 2^31 range of the high words (|w| ~ 1e30)
    keep the fp32-atomic path (f32_fixed_bits = -1), still within T2."""
    n_rows, n_cols = 2000, 40_000
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.05, seed=12, weights="uniform",
                                    w0=-1e30, w1=1e30)
    tip, tix, tdat = _t(ip), _t(ix), _t(dat)
    plan = bp.csrmv_plan(tip, tix, n_rows, n_cols, torch.float32, homo=False, data=tdat)
    assert plan is not None and plan.f32_fixed_bits == -1
    ev = inputs.spike_pattern(n_rows, 0.2, 5)
    out = torch.zeros(n_cols, dtype=torch.float32, device="cuda")
    bp.event_csrmv(tip, tix, tdat, 0.0, n_rows, n_cols, _dev_spikes(ev), out, plan=plan)
    ref, absw = orc.event_csrmv(ip, ix, dat, 0.0, n_rows, n_cols, ev, orc.OUT_F64, with_abs=True)
    err = np.abs(out.cpu().numpy().astype(np.float64) - ref)
    assert np.all(err <= 1e-5 * absw + 1e-30)
