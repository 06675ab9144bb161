"""GPU parity of the geometric-gap sampler (rule J10; SURVEY 8(f)
NEXT 4) against the CPU oracle.

Positions and every BP_OUT_FIX64 output are bit-exact (both sides draw the
same gaps through the op-for-op specified fp32 log of rule J10); BP_OUT_F32
outputs satisfy rule T2.  Normal-law weights are bit-identical too (J7n).
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


def _specs(bp, orc, seed, p, seg_len, n_cols, law="homo", w0=0.6, w1=0.0):
    L = seg_len or n_cols
    ospec = orc.JitSpec(seed, orc.conn_len(p), L, orc.LAWS[law], w0, w1, geo_c=orc.geo_c(p))
    return bp.jitconn_spec(seed, p, 0, seg_len, gap_law=bp.GAP_GEOMETRIC), ospec


@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
@pytest.mark.parametrize("shape", [(200, 5000, 0.05, 0), (100, 4000, 0.1, 300),
                                   (50, 37, 1.0, 0), (40, 20_000, 0.0004, 0),
                                   (300, 1000, 0.5, 100)])
def test_geo_materialize_bit_exact(bp, orc, law, shape):
    n_rows, n_cols, p, seg_len = shape
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-1.0, 1.0), "normal": (0.5, 2.0)}[law]
    spec, ospec = _specs(bp, orc, 4243, p, seg_len, n_cols, law, w0, w1)
    ip, ix, dat = bp.jitconn_materialize(spec, n_rows, n_cols, law=orc.LAWS[law], w0=w0, w1=w1)
    oip, oix, odat = orc.jit_materialize(ospec, n_rows, n_cols)
    assert np.array_equal(ip.cpu().numpy(), oip)
    assert np.array_equal(ix.cpu().numpy(), oix)
    dat = dat.cpu().numpy()
    assert np.array_equal(dat.view(np.uint32), odat.view(np.uint32))   # J7n: every law


def test_geo_differs_from_uniform_and_has_density_p(bp, orc):
    """Same seed, other sampler: another matrix, of density p (not 2/(K+1))."""
    n_rows, n_cols, p = 2000, 2000, 0.03          # K = 65, 2/(K+1) = 0.0303
    spec, _ = _specs(bp, orc, 5, p, 0, n_cols)
    ip, ix, _ = bp.jitconn_materialize(spec, n_rows, n_cols, with_data=False)
    ipu, ixu, _ = bp.jitconn_materialize(bp.jitconn_spec(5, p), n_rows, n_cols,
                                         with_data=False)
    assert not torch.equal(ip, ipu)
    cells = n_rows * n_cols
    assert abs(int(ip[-1]) - cells * p) < 4 * np.sqrt(cells * p * (1 - p))


JIT_CASES = [
    # n_rows, n_cols, p, seg_len, density
    (64, 37, 1.0, 0, 0.5),             # p = 1: dense rows
    (500, 3000, 0.05, 0, 0.1),
    (300, 10_000, 0.1, 1000, 0.2),     # 10 segments
    (1000, 100_000, 0.05, 0, 0.01),    # config-2 row shape, tiled path
    (200, 300_000, 0.005, 0, 0.1),     # many column tiles
    (3000, 20_000, 0.0005, 0, 0.3),    # sparse rows (~10 targets)
]


@pytest.mark.parametrize("path", ["tiled", "direct"])
@pytest.mark.parametrize("case", JIT_CASES)
@pytest.mark.parametrize("law", ["homo", "uniform", "normal"])
def test_geo_event_mv(bp, orc, case, law, path, monkeypatch):
    monkeypatch.setenv("BP_JIT_DIRECT" if path == "direct" else "BP_JIT_TILED", "1")
    n_rows, n_cols, p, seg_len, density = case
    w0, w1 = {"homo": (0.6, 0.0), "uniform": (-0.1, 0.1), "normal": (0.0, 0.3)}[law]
    seed = 0xBEEF + n_rows
    spec, ospec = _specs(bp, orc, seed, p, seg_len, n_cols, law, w0, w1)
    ev = inputs.spike_pattern(n_rows, density, seed=19)
    spikes = _dev_spikes(ev)
    fn = {"homo": lambda o: bp.jitconn_event_mv_homo(spec, w0, spikes, n_rows, n_cols, o),
          "uniform": lambda o: bp.jitconn_event_mv_uniform(spec, w0, w1, spikes, n_rows,
                                                           n_cols, o),
          "normal": lambda o: bp.jitconn_event_mv_normal(spec, w0, w1, spikes, n_rows,
                                                         n_cols, o)}[law]
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


@pytest.mark.parametrize("bounds", [(0, 1000), (1000, 5000), (9000, 10_000)])
def test_geo_partition(bp, orc, bounds):
    n_rows, n_cols, L = 400, 10_000, 1000
    cb, ce = bounds
    spec, ospec = _specs(bp, orc, 78, 0.02, L, n_cols, "uniform", -1.0, 1.0)
    ev = inputs.spike_pattern(n_rows, 0.3, seed=4)
    out = torch.zeros(ce - cb, dtype=torch.int64, device="cuda")
    bp.jitconn_event_mv_uniform(spec, -1.0, 1.0, _dev_spikes(ev), n_rows, n_cols, out,
                                col_begin=cb, col_end=ce)
    want = orc.jit_event_mv(ospec, n_rows, n_cols, ev, cb, ce, orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want)


@pytest.mark.parametrize("path", ["tiled", "direct"])
def test_geo_mv(bp, orc, path, monkeypatch):
    """Non-event product over the geometric matrix (reading MV1)."""
    monkeypatch.setenv("BP_JIT_DIRECT" if path == "direct" else "BP_JIT_TILED", "1")
    n_rows, n_cols, p = 300, 100_000, 0.05
    spec, ospec = _specs(bp, orc, 31, p, 0, n_cols, "uniform", -0.1, 0.2)
    rng = np.random.default_rng(3)
    v = rng.normal(0.0, 2.0, n_rows).astype(np.float32)
    v[rng.random(n_rows) < 0.3] = 0.0
    out = torch.zeros(n_cols, dtype=torch.int64, device="cuda")
    bp.jitconn_mv(bp.LAW_UNIFORM, spec, -0.1, 0.2, torch.from_numpy(v).cuda(), n_rows,
                  n_cols, out)
    want = orc.jit_mv(ospec, n_rows, n_cols, v, out_kind=orc.OUT_FIX)
    assert np.array_equal(out.cpu().numpy(), want)


def test_geo_errors(bp):
    out = torch.zeros(1000, device="cuda")
    sp = _dev_spikes(np.ones(10, np.uint8))
    # positions would exceed 32 bits: n_cols + 128 (L + 1) >= 2^32
    big = bp.jitconn_spec(1, 0.5, 0, 0, gap_law=bp.GAP_GEOMETRIC)
    with pytest.raises(bp.BpError, match="UNSUPPORTED"):
        bp.jitconn_event_mv_homo(big, 1.0, sp, 10, 40_000_000,
                                 torch.zeros(40_000_000, device="cuda"))
    bad = bp.jitconn_spec(1, 0.1, 0, 0, gap_law=7)
    with pytest.raises(bp.BpError, match="INVALID"):
        bp.jitconn_event_mv_homo(bad, 1.0, sp, 10, 1000, out)
    # networks run the uniform sampler only
    from paper_2311_05106_b200.network import CobaNetwork
    net = CobaNetwork(4000, fixed=True, device="cuda")
    spec = bp.jitconn_spec(1, 0.02, 0, 0, gap_law=bp.GAP_GEOMETRIC)
    with pytest.raises(bp.BpError, match="UNSUPPORTED"):
        bp.Network(model=bp.MODEL_LIF, n=4000, state=net.state, spikes=net.spikes,
                   params=net.params, col_begin=0, col_end=4000,
                   projections=[bp.projection(pre_begin=0, pre_end=3200, weight=0.6, jit=spec),
                                bp.projection(pre_begin=3200, pre_end=4000, weight=6.7,
                                              receptor=bp.RECEPTOR_INH, jit=spec)])
