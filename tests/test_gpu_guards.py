"""Out-of-bounds write checks of every libbp kernel family with guard
regions (compute-sanitizer is not available on the GPU pool): every buffer a
call writes -- outputs, network state, spike vectors, rasters, workspaces --
is a view into a larger allocation whose head and tail (1 KB each) hold a
random pattern, and the pattern must survive the calls.  Plus the debug NaN
check of the network (BP_DEBUG_NAN=1: the SPEC's NaN abort as a
device counter)."""
import numpy as np
import pytest
import torch

import paper_2311_05106_b200 as bp
from paper_2311_05106_b200 import inputs

pytestmark = pytest.mark.gpu
GUARD_BYTES = 1024


@pytest.fixture(scope="module", autouse=True)
def _built():
    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)


class Guards:
    """Allocates guarded views and checks every guard at the end."""

    def __init__(self):
        self.bufs = []
        self.gen = torch.Generator(device="cuda").manual_seed(1234)

    def __call__(self, n, dtype, fill=None):
        item = torch.empty(0, dtype=dtype).element_size()
        g = GUARD_BYTES // item
        full = torch.empty(n + 2 * g, dtype=dtype, device="cuda")
        raw = full.view(torch.uint8)
        raw.copy_(torch.randint(0, 256, raw.shape, generator=self.gen, device="cuda",
                                dtype=torch.int32).to(torch.uint8))
        view = full[g:g + n]
        if fill is not None:
            view.copy_(torch.as_tensor(fill).to(dtype))
        # guards compared as raw bytes (a random float pattern may be a NaN)
        self.bufs.append((full, g, n, full[:g].view(torch.uint8).clone(),
                          full[g + n:].view(torch.uint8).clone()))
        return view

    def check(self):
        torch.cuda.synchronize()
        for k, (full, g, n, head, tail) in enumerate(self.bufs):
            assert torch.equal(full[:g].view(torch.uint8), head), \
                f"buffer {k}: write before the start"
            assert torch.equal(full[g + n:].view(torch.uint8), tail), \
                f"buffer {k}: write past the end"


def test_stateless_kernels_write_only_their_outputs():
    G = Guards()
    n_rows, n_cols = 3000, 2500
    ev = inputs.spike_pattern(n_rows, 0.1, 1)
    spikes = G(inputs.n_words(n_rows), torch.int32,
               torch.from_numpy(inputs.pack_bits(ev).view(np.int32)))
    active = G(n_rows, torch.int32)
    count = G(1, torch.int32)
    bp.compact_spikes(spikes, n_rows, active, count)
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.05, seed=5, weights="uniform", w0=-1, w1=1)
    tip, tix, tdat = (torch.from_numpy(a).cuda() for a in (ip, ix, dat))
    for dtype, kind in ((torch.float32, 0), (torch.int64, 1)):
        for data in (tdat, None):
            out = G(n_cols, dtype)
            ws = G(int(bp.lib().bp_csrmv_workspace_bytes(n_rows, n_cols, kind)), torch.uint8)
            bp.event_csrmv(tip, tix, data, 0.5, n_rows, n_cols, spikes, out, ws=ws)
            plan = bp.csrmv_plan(tip, tix, n_rows, n_cols, dtype, homo=data is None, data=data)
            bp.event_csrmv(tip, tix, data, 0.5, n_rows, n_cols, spikes, out, ws=ws, plan=plan)
            small = G(bp.workspace_bytes(n_rows), torch.uint8)      # per-event fallback
            bp.event_csrmv(tip, tix, data, 0.5, n_rows, n_cols, spikes, out, ws=small)
        sp_cols = G(inputs.n_words(n_cols), torch.int32, torch.from_numpy(
            inputs.pack_bits(inputs.spike_pattern(n_cols, 0.1, 2)).view(np.int32)))
        bp.csrmv_gather(tip, tix, tdat, 0.5, n_rows, n_cols, sp_cols, G(n_rows, dtype))
    gy = torch.randn(n_cols, device="cuda")
    gw = G(1, torch.float64)
    bp.event_csrmv_grad(tip, tix, tdat, 0.5, n_rows, n_cols, spikes, gy, G(tix.numel(), torch.float32),
                        G(n_rows, torch.float32), None)
    bp.event_csrmv_grad(tip, tix, None, 0.5, n_rows, n_cols, spikes, gy, None,
                        G(n_rows, torch.float32), gw)
    for p in (0.05, 0.5):
        for gap in (bp.GAP_UNIFORM, bp.GAP_GEOMETRIC):
            spec = bp.jitconn_spec(7, p, gap_law=gap)
            for dtype, kind in ((torch.float32, 0), (torch.int64, 1)):
                for c0, c1 in ((0, n_cols), (0, 1250), (1250, n_cols)):
                    sspec = bp.jitconn_spec(7, p, seg_len=1250, gap_law=gap)
                    use = spec if (c0, c1) == (0, n_cols) else sspec
                    out = G(c1 - c0, dtype)
                    ws = G(int(bp.lib().bp_jitconn_workspace_bytes(n_rows, c0, c1, kind)),
                           torch.uint8)
                    for law, w0, w1 in ((bp.LAW_HOMO, 0.6, 0.0), (bp.LAW_UNIFORM, -0.1, 0.1),
                                        (bp.LAW_NORMAL, 0.0, 0.1)):
                        bp.jitconn_event_mv(law, use, w0, w1, spikes, n_rows, n_cols, out,
                                            col_begin=c0, col_end=c1, ws=ws)
                        v = torch.randn(n_rows, device="cuda")
                        bp.jitconn_mv(law, use, w0, w1, v, n_rows, n_cols, out, col_begin=c0,
                                      col_end=c1, ws=ws)
    n = 5000
    for model, params in ((bp.MODEL_LIF, bp.lif_params()), (bp.MODEL_HH, bp.hh_params())):
        for g_dtype in (torch.float32, torch.int64, torch.int32):
            st = {"v": G(n, torch.float32, -60.0), "g_e": G(n, g_dtype, 0),
                  "g_i": G(n, g_dtype, 0)}
            if model == bp.MODEL_LIF:
                st["ref"] = G(n, torch.uint8, 0)
            else:
                for k in ("m", "h", "n"):
                    st[k] = G(n, torch.float32, 0.3)
            bp.neuron_step(params, st, G(inputs.n_words(n), torch.int32), G(n, torch.int32),
                           G(1, torch.int32, 0))
    G.check()


def _guarded_network(G, n, g_dtype, *, model="lif", delay=1, merged=False, exchange=None):
    p = 80.0 / n
    n_exc = n * 4 // 5
    st = {"g_e": G(n, g_dtype, 0), "g_i": G(n, g_dtype, 0)}
    if g_dtype == torch.int32:
        st["frac_bits"] = 20 if model == "lif" else 16
    if model == "lif":
        st["v"] = G(n, torch.float32, torch.from_numpy(inputs.lif_v0(n)))
        st["ref"] = G(n, torch.uint8, 0)
        params = bp.lif_params()
        w = (0.6, 6.7)
    else:
        v, m, h, nk = inputs.hh_init(n)
        for k, a in (("v", v), ("m", m), ("h", h), ("n", nk)):
            st[k] = G(n, torch.float32, torch.from_numpy(a))
        params = bp.hh_params()
        w = (6.0, 67.0)
    spikes = G(inputs.n_words(n), torch.int32, 0)
    K = bp.conn_len(p)
    if merged:
        cuts = [(0, n_exc // 3, 0, 0.6), (n_exc // 3, n_exc, 0, 0.45), (n_exc, n, 1, 6.7)]
    else:
        cuts = [(0, n_exc, 0, w[0]), (n_exc, n, 1, w[1])]
    projs = [bp.projection(pre_begin=b, pre_end=e, weight=ww, receptor=r,
                           jit=bp.jitconn_spec(0x5EED0001 + k, p, K, n))
             for k, (b, e, r, ww) in enumerate(cuts)]
    kw = {}
    if exchange == "nccl":
        kw = dict(exchange=bp.EXCHANGE_NCCL, rank=0, world=1, part_len=(n + 31) // 32 * 32,
                  nccl_id=bp.nccl_unique_id())
    probe = bp.Network(model=bp.MODEL_LIF if model == "lif" else bp.MODEL_HH, n=n, state=st,
                       spikes=spikes, params=params, projections=projs, delay=delay, **kw)
    ws = G(probe.ws.numel(), torch.uint8, 0)
    probe.close()
    if exchange == "nccl":
        kw["nccl_id"] = bp.nccl_unique_id()          # an NCCL id serves one communicator
    return bp.Network(model=bp.MODEL_LIF if model == "lif" else bp.MODEL_HH, n=n, state=st,
                      spikes=spikes, params=params, projections=projs, delay=delay, ws=ws, **kw)


@pytest.mark.parametrize("case", ["small", "tiles_f32", "tiles_fix32_delay3", "hh_dense",
                                  "merged_fix64", "nccl_delay2"])
def test_network_kernels_write_only_their_buffers(case, monkeypatch):
    G = Guards()
    n, dt, kw = {"small": (4000, torch.int64, {}),
                 "tiles_f32": (20_000, torch.float32, {}),
                 "tiles_fix32_delay3": (20_000, torch.int32, {"delay": 3}),
                 "hh_dense": (12_000, torch.float32, {"model": "hh"}),
                 "merged_fix64": (20_000, torch.int64, {"merged": True}),
                 "nccl_delay2": (20_000, torch.int64, {"delay": 2, "exchange": "nccl"})}[case]
    net = _guarded_network(G, n, dt, **kw)
    steps = 60
    raster = G(steps * net.local_words, torch.int32).view(steps, net.local_words)
    counts = G(steps, torch.int32)
    net.step(steps // 2, raster[:steps // 2], counts[:steps // 2])
    net.step(steps - steps // 2, raster[steps // 2:], counts[steps // 2:])
    G.check()
    assert int(counts.sum().item()) > 0


def test_debug_nan_check_counts_nonfinite_potentials(monkeypatch):
    """BP_DEBUG_NAN=1: a NaN membrane potential is counted after every step
    (it stays NaN: the update propagates it); a clean run counts 0."""
    from paper_2311_05106_b200.network import CobaNetwork
    monkeypatch.setenv("BP_DEBUG_NAN", "1")
    monkeypatch.setenv("BP_NO_SMALL_NET", "1")
    clean = CobaNetwork(8000, conn="jit", fixed=False)
    clean.run(50)
    assert clean.net.counters_all()[3] == 0
    v0 = inputs.lif_v0(8000)
    v0[[3, 4000, 7999]] = np.nan
    bad = CobaNetwork(8000, conn="jit", fixed=False, v0=v0)
    bad.run(50)
    assert bad.net.counters_all()[3] >= 3 * 50
