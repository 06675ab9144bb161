"""Pins for the oracle's network loop (rule S1, Listing S3 update()).

* A w = 0 network is a set of unconnected LIF neurons: each raster row has a
  closed form (first passage from V0, then period 189 steps).
* Fixed-point g after T steps equals the fp64 recursion
  g_n = alpha g_{n-1} + sum_{r in spikes_{n-1}} w D[r, c] recomputed in
  numpy from the oracle's own raster and an independent densified matrix,
  within the F1 rounding bound.
* The JIT network equals the network over its materialised CSR.
* Refractory contract and determinism.
Firing *rates* of the coupled network are not printed in the paper
(Fig 2C elided): parity for rates is unpinned (reading R23).
"""
import math

import numpy as np
import pytest

from paper_2311_05106_b200 import inputs


def _coba(orc, n=4000, fixed=True, w_e=0.6, w_i=6.7, seed_e=0x5EED0001,
          seed_i=0x5EED0002, conn="jit"):
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(seed_e, K, n, orc.LAW_HOMO, w_e))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(seed_i, K, n, orc.LAW_HOMO, w_i))
    if conn == "csr":
        ip, ix, _ = orc.jit_materialize(pe.jit, n_exc, n)
        pe = orc.Projection(0, n_exc, csr=(ip, ix, None), w_homo=w_e)
        ip, ix, _ = orc.jit_materialize(pi.jit, n - n_exc, n)
        pi = orc.Projection(n_exc, n - n_exc, csr=(ip, ix, None), w_homo=w_i)
    g_dtype = np.int64 if fixed else np.float32
    state = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, g_dtype),
                 g_i=np.zeros(n, g_dtype), ref=np.zeros(n, np.uint8),
                 spikes=np.zeros(n, np.uint8))
    return state, pe, pi


def test_zero_weight_network_closed_form(orc):
    n = 800
    state, pe, pi = _coba(orc, n=n, w_e=0.0, w_i=0.0)
    v0 = state["v"].astype(np.float64).copy()
    raster = orc.run_network("lif", orc.lif_params(), state, pe, pi, 700)
    alpha = math.exp(-0.1 / 20.0)
    checked = 0
    for i in range(n):
        # V_m = -40 + (V0 + 40) alpha^m; first m >= 1 with V_m > -50
        ratio = 10.0 / (-40.0 - v0[i])
        m_real = math.log(ratio) / math.log(alpha) if ratio < 1 else 0.0
        if abs(m_real - round(m_real)) < 0.05:
            continue          # fp32 rounding could move a near-integer crossing
        m1 = max(1, math.floor(m_real) + 1)
        want = list(range(m1 - 1, 700, 189))
        got = np.nonzero(raster[:, i])[0].tolist()
        assert got == want, i
        checked += 1
    assert checked > 700


def test_fixed_point_g_equals_fp64_recursion(orc):
    n, T = 4000, 300
    state, pe, pi = _coba(orc, n=n)
    raster = orc.run_network("lif", orc.lif_params(), state, pe, pi, T)
    assert raster.sum() > 0
    # independent dense matrices from the oracle's materialised rows
    d_e = np.zeros((pe.n_rows, n))
    for r in range(pe.n_rows):
        d_e[r, orc.jit_row(pe.jit, n, r)[0]] = float(np.float32(0.6))
    d_i = np.zeros((pi.n_rows, n))
    for r in range(pi.n_rows):
        d_i[r, orc.jit_row(pi.jit, n, r)[0]] = float(np.float32(6.7))
    a_e, a_i = math.exp(-0.1 / 5.0), math.exp(-0.1 / 10.0)
    g_e = np.zeros(n); g_i = np.zeros(n)
    prev = np.zeros(n)
    for step in range(T):
        g_e = a_e * g_e + prev[:pe.n_rows] @ d_e      # decay, then add (R12)
        g_i = a_i * g_i + prev[pe.n_rows:] @ d_i
        prev = raster[step].astype(np.float64)
    # the stored state is pre-decayed after the last update
    g_e *= a_e
    g_i *= a_i
    got_e = state["g_e"] / 2.0 ** 32
    got_i = state["g_i"] / 2.0 ** 32
    # per step <= 1 unit of 2^-32 from llrint(decay) + 0.5/term: << 2^-20
    assert np.max(np.abs(got_e - g_e)) < 2.0 ** -20 * max(1.0, g_e.max())
    assert np.max(np.abs(got_i - g_i)) < 2.0 ** -20 * max(1.0, g_i.max())


def test_fix32_g_within_bound_of_fp64_recursion(orc):
    """Rule F2 (int32, F = 20 fractional bits): the conductance stays within
    the accumulated rounding bound of the exact recursion."""
    n, T, F = 4000, 300, 20
    orc.set_fix32_bits(F)
    state, pe, pi = _coba(orc, n=n)
    state["g_e"] = np.zeros(n, np.int32)
    state["g_i"] = np.zeros(n, np.int32)
    raster = orc.run_network("lif", orc.lif_params(), state, pe, pi, T)
    assert raster.sum() > 0
    d_e = np.zeros((pe.n_rows, n))
    for r in range(pe.n_rows):
        d_e[r, orc.jit_row(pe.jit, n, r)[0]] = float(np.float32(0.6))
    d_i = np.zeros((pi.n_rows, n))
    for r in range(pi.n_rows):
        d_i[r, orc.jit_row(pi.jit, n, r)[0]] = float(np.float32(6.7))
    a_e, a_i = math.exp(-0.1 / 5.0), math.exp(-0.1 / 10.0)
    g_e = np.zeros(n); g_i = np.zeros(n); prev = np.zeros(n)
    events_e = np.zeros(n); events_i = np.zeros(n)
    for step in range(T):
        inc_e = prev[:pe.n_rows] @ (d_e > 0)
        inc_i = prev[pe.n_rows:] @ (d_i > 0)
        events_e = np.maximum(events_e, inc_e)
        events_i = np.maximum(events_i, inc_i)
        g_e = a_e * g_e + prev[:pe.n_rows] @ d_e
        g_i = a_i * g_i + prev[pe.n_rows:] @ d_i
        prev = raster[step].astype(np.float64)
    g_e *= a_e
    g_i *= a_i
    # per step: <= 1/2 ulp from the decay + 1/2 ulp per quantised event;
    # errors contract by alpha, so the stationary bound is that / (1 - alpha)
    ulp = 2.0 ** -F
    bound_e = (0.5 + 0.5 * events_e.max()) * ulp / (1 - a_e) + ulp
    bound_i = (0.5 + 0.5 * events_i.max()) * ulp / (1 - a_i) + ulp
    assert np.max(np.abs(state["g_e"] * ulp - g_e)) <= bound_e
    assert np.max(np.abs(state["g_i"] * ulp - g_i)) <= bound_i
    orc.set_fix32_bits(20)


def test_fix32_saturation(orc):
    g = np.array([2 ** 31 - 10, -(2 ** 31) + 5, 7], np.int32)
    sat = orc.fix32_add(g, np.array([100, -100, 3], np.int64))
    assert sat == 2
    assert g.tolist() == [2 ** 31 - 1, -(2 ** 31), 10]


def test_jit_network_equals_materialised_csr_network(orc):
    n, T = 2000, 200
    s1, pe1, pi1 = _coba(orc, n=n)
    s2, pe2, pi2 = _coba(orc, n=n, conn="csr")
    r1 = orc.run_network("lif", orc.lif_params(), s1, pe1, pi1, T)
    r2 = orc.run_network("lif", orc.lif_params(), s2, pe2, pi2, T)
    assert np.array_equal(r1, r2)
    assert np.array_equal(s1["v"].view(np.uint32), s2["v"].view(np.uint32))
    assert np.array_equal(s1["g_e"], s2["g_e"])


def test_refractory_contract_and_determinism(orc):
    n, T = 4000, 400
    s1, pe, pi = _coba(orc, n=n)
    r1 = orc.run_network("lif", orc.lif_params(), s1, pe, pi, T)
    s2, pe, pi = _coba(orc, n=n)
    r2 = orc.run_network("lif", orc.lif_params(), s2, pe, pi, T)
    assert np.array_equal(r1, r2)
    for i in range(n):
        t = np.nonzero(r1[:, i])[0]
        assert np.all(np.diff(t) >= 51)


@pytest.mark.parametrize("fixed", [True, False])
def test_hh_network_runs_finite(orc, fixed):
    n = 1000
    n_exc = 800
    K = orc.conn_len(80.0 / n)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(1, K, n, orc.LAW_HOMO, 6.0))
    pi = orc.Projection(n_exc, n - n_exc, jit=orc.JitSpec(2, K, n, orc.LAW_HOMO, 67.0))
    v, m, h, nk = inputs.hh_init(n)
    g_dtype = np.int64 if fixed else np.float32
    state = dict(v=v, m=m, h=h, n=nk, g_e=np.zeros(n, g_dtype),
                 g_i=np.zeros(n, g_dtype), spikes=np.zeros(n, np.uint8))
    raster = orc.run_network("hh", orc.hh_params(), state, pe, pi, 300)
    assert np.all(np.isfinite(state["v"]))
    assert raster.sum() > 0


# ---------------------------------------------------------------- reading D1
@pytest.mark.parametrize("delay", [1, 3, 8])
def test_delay_single_spike_arrives_after_d_steps(orc, delay):
    """One presynaptic spike in spikes_{-1}, a network that stays silent on
    its own: the spike's targets receive w at step D-1 (0-based) and decay
    afterwards; nothing arrives before.  Fixed point (F1) makes it exact."""
    n, T = 400, 12
    state, pe, pi = _coba(orc, n=n)
    state["v"][:] = -60.0                    # rest: first own spike after 139 steps
    state["spikes"][:] = 0
    state["spikes"][5] = 1                   # excitatory row 5
    targets = orc.jit_row(pe.jit, n, 5)[0]
    for t_end in (delay - 1, delay, T):      # before / just after / well after delivery
        st = {k: (v.copy() if hasattr(v, "copy") else v) for k, v in state.items()}
        raster = orc.run_network("lif", orc.lif_params(), st, pe, pi, t_end, delay=delay)
        assert raster.sum() == 0
        g = st["g_e"]
        if t_end < delay:
            assert not g.any()
            continue
        # delivered at step delay-1, then decayed (t_end - delay + 1) times
        # by rule F1: g <- llrint(g * alpha_E) in fp64
        alpha = math.exp(-0.1 / 5.0)
        want = int(orc.quantize(np.float32(0.6)))
        for _ in range(t_end - delay + 1):
            want = int(np.rint(np.float64(want) * alpha))
        assert np.all(g[targets] == want), (t_end, g[targets][:3], want)
        others = np.setdiff1d(np.arange(n), targets)
        assert not g[others].any()


def test_delay_one_equals_default_and_history_continues(orc):
    """delay = 1 is rule S1; a delayed run split in two calls equals one call."""
    n, T = 2000, 120
    s1, pe, pi = _coba(orc, n=n)
    r1 = orc.run_network("lif", orc.lif_params(), s1, pe, pi, T)
    s2, _, _ = _coba(orc, n=n)
    r2 = orc.run_network("lif", orc.lif_params(), s2, pe, pi, T, delay=1)
    assert np.array_equal(r1, r2)
    s3, _, _ = _coba(orc, n=n)
    ra = orc.run_network("lif", orc.lif_params(), s3, pe, pi, 50, delay=4)
    rb = orc.run_network("lif", orc.lif_params(), s3, pe, pi, T - 50, delay=4)
    s4, _, _ = _coba(orc, n=n)
    rc = orc.run_network("lif", orc.lif_params(), s4, pe, pi, T, delay=4)
    assert np.array_equal(np.vstack([ra, rb]), rc)
    assert not np.array_equal(rc, r1)        # the delay changes the dynamics


# ---------------------------------------------------------------- rule N1-f32
# The fp32 conductance mode (the bench's default): a homogeneous projection
# delivers `count` identical weights to a neuron in one step and the
# increment is fl32(count * w), the exactly rounded sum (N1-f32);
# then g <- fl32(g + inc), the neuron reads g, and g <- fl32(g * fl32(alpha))
# (Expon: decay, then add -- reading R12).

def _round_f32_exact(q):
    """Round the exact rational q to the nearest float32 (ties to even),
    independently of any fp32 arithmetic: bracket q between the two float32
    neighbours of float64(q) and pick the nearer one with Fractions."""
    from fractions import Fraction
    x = np.float32(float(q))
    cands = [np.nextafter(x, np.float32(-np.inf)), x, np.nextafter(x, np.float32(np.inf))]
    best = min(cands, key=lambda c: (abs(Fraction(float(c)) - q),
                                     int(np.array(c, np.float32).view(np.uint32)) & 1))
    return np.float32(best)


def test_f32_increment_is_the_exactly_rounded_sum(orc):
    """A neuron receiving k events of w = fl32(0.6) in one step gets exactly
    round_f32(k * w) (exact rational arithmetic), which for some k differs
    from summing the k weights one by one in fp32 -- so the oracle's rule is
    the exactly rounded sum, not a sequential fp32 accumulation."""
    from fractions import Fraction
    w = np.float32(0.6)
    differs = 0
    for k in (1, 2, 3, 7, 10, 13, 37, 80, 129, 1000):
        n = k + 32
        ip = np.zeros(n + 1, np.int64)
        ip[1:k + 1] = np.arange(1, k + 1)            # rows 0..k-1 -> column 0
        ip[k + 1:] = k
        ix = np.zeros(k, np.int32)
        pe = orc.Projection(0, n, csr=(ip, ix, None), w_homo=float(w))
        pi = orc.Projection(n, 0, csr=(np.zeros(1, np.int64), np.zeros(0, np.int32), None),
                            w_homo=6.7)
        spikes = np.zeros(n, np.uint8)
        spikes[:k] = 1
        st = dict(v=np.full(n, -60.0, np.float32), g_e=np.zeros(n, np.float32),
                  g_i=np.zeros(n, np.float32), ref=np.zeros(n, np.uint8), spikes=spikes)
        # tau_E = inf: alpha = 1, so the stored g is the increment itself
        orc.run_network("lif", orc.lif_params(tau_e=float("inf")), st, pe, pi, 1)
        want = _round_f32_exact(k * Fraction(float(w)))
        assert st["g_e"][0].view(np.uint32) == want.view(np.uint32), k
        assert np.all(st["g_e"][1:] == 0)
        seq = np.float32(0)
        for _ in range(k):
            seq = np.float32(seq + w)
        differs += int(seq != want)
    assert differs > 0          # the pin distinguishes the two summation rules


def test_f32_g_within_bound_of_fp64_recursion(orc):
    """Rule N1-f32 over 300 steps of the 4000-neuron network: the fp32 g
    equals the exact fp64 recursion a_n = alpha a_{n-1} + inc_n (recomputed
    from the oracle's raster with an independent dense matrix) within the
    rounding bound of the fp32 rule.  With u = 2^-24, per step
      |err_n| <= alpha |err_{n-1}| + |alpha32 - alpha| |a_{n-1}|
                 + u (|alpha a_{n-1}| + |inc_n| + |a_n|)      (+ 1 % slack),
    the three roundings being the decay product, fl32(count w) and the add.
    A dropped or misplaced term (add after the decay, w of the other
    projection, alpha of the other synapse) moves g by far more."""
    n, T = 4000, 300
    state, pe, pi = _coba(orc, n=n, fixed=False)
    raster = orc.run_network("lif", orc.lif_params(), state, pe, pi, T)
    assert raster.sum() > 0
    u = 2.0 ** -24
    out = []
    for proj, w, tau, rows in ((pe, 0.6, 5.0, slice(0, pe.n_rows)),
                               (pi, 6.7, 10.0, slice(pe.n_rows, n))):
        d = np.zeros((proj.n_rows, n))
        for r in range(proj.n_rows):
            d[r, orc.jit_row(proj.jit, n, r)[0]] = float(np.float32(w))
        a = math.exp(-0.1 / tau)
        a32 = float(np.float32(a))
        g = np.zeros(n)
        b = np.zeros(n)
        prev = np.zeros(n)
        for step in range(T):
            inc = prev[rows] @ d
            g_new = a * g + inc                        # decay, then add (R12)
            b = a * b + abs(a32 - a) * g + u * (a * g + inc + g_new)
            g = g_new
            prev = raster[step].astype(np.float64)
        # stored state: pre-decayed once more
        b = a * b + abs(a32 - a) * g + u * a * g
        g = a * g
        out.append((g, b * 1.01 + 1e-30))
    (ge, be), (gi, bi) = out
    err_e = np.abs(state["g_e"].astype(np.float64) - ge)
    err_i = np.abs(state["g_i"].astype(np.float64) - gi)
    assert np.all(err_e <= be), float(np.max(err_e - be))
    assert np.all(err_i <= bi), float(np.max(err_i - bi))
    # the bound is tight enough to matter: well below one event's weight
    assert be.max() < 1e-3 * 0.6 and bi.max() < 1e-3 * 6.7


@pytest.mark.parametrize("g_dtype", [np.int64, np.int32, np.float32])
def test_threaded_oracle_equals_sequential(orc, g_dtype):
    """The oracle's optional host threads (order-free loops only: per-neuron
    updates and integer event scatters) give bit-identical networks."""
    n, T = 4000, 150
    runs = []
    for threads in (1, 4):
        orc.set_threads(threads)
        try:
            state, pe, pi = _coba(orc, n=n)
            state["g_e"] = np.zeros(n, g_dtype)
            state["g_i"] = np.zeros(n, g_dtype)
            raster = orc.run_network("lif", orc.lif_params(), state, pe, pi, T)
        finally:
            orc.set_threads(1)
        runs.append((raster, state))
    (r1, s1), (r2, s2) = runs
    assert r1.sum() > 0 and np.array_equal(r1, r2)
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(s1[k].view(np.uint8), s2[k].view(np.uint8)), k


# ------------------------------------------------- AlignPost merging
# Several projections into one receptor share its single conductance per
# neuron; the step's increment is the exact sum of all their events
# (fixed point) or its exactly rounded value (rule N1-f32).

def _split_csr(ip, ix, cut):
    """Rows [0, cut) and [cut, n_rows) of a CSR as two CSRs."""
    a = (ip[:cut + 1].copy(), ix[:ip[cut]].copy(), None)
    b = ((ip[cut:] - ip[cut]).copy(), ix[ip[cut]:].copy(), None)
    return a, b


@pytest.mark.parametrize("g_dtype", [np.int64, np.int32, np.float32])
def test_merged_projections_equal_their_union(orc, g_dtype):
    """Listing S3's E projection cut into two projections over rows
    [0, 1000) and [1000, 3200) with the same weight, both adding into g_E,
    is the same network: rasters and state bit for bit in every mode."""
    n, T = 4000, 200
    s1, pe, pi = _coba(orc, n=n, conn="csr")
    s1["g_e"] = np.zeros(n, g_dtype)
    s1["g_i"] = np.zeros(n, g_dtype)
    r1 = orc.run_network("lif", orc.lif_params(), s1, pe, pi, T)
    s2, _, _ = _coba(orc, n=n, conn="csr")
    s2["g_e"] = np.zeros(n, g_dtype)
    s2["g_i"] = np.zeros(n, g_dtype)
    (a, b) = _split_csr(*pe.csr[:2], 1000)
    projs = [orc.Projection(0, 1000, csr=a, w_homo=0.6, receptor="exc"),
             orc.Projection(1000, pe.n_rows - 1000, csr=b, w_homo=0.6, receptor="exc"),
             orc.Projection(pi.row0, pi.n_rows, csr=pi.csr, w_homo=6.7, receptor="inh")]
    r2 = orc.run_network("lif", orc.lif_params(), s2, projs, None, T)
    assert r1.sum() > 0 and np.array_equal(r1, r2)
    for k in ("v", "g_e", "g_i", "ref"):
        assert np.array_equal(s1[k].view(np.uint8), s2[k].view(np.uint8)), k


def test_merged_distinct_weights_fixed_point_recursion(orc):
    """Two excitatory projections with different weights (0.6 and 0.45,
    different JIT seeds) and one inhibitory, merged: the fixed-point g_E
    equals the fp64 recursion a_n = alpha a_{n-1} + sum_p w_p D_p^T s_{n-1}
    from the raster and independent dense matrices, within the F1 bound."""
    n, T, n1 = 3000, 250, 1200
    n_exc = n * 4 // 5
    K = orc.conn_len(80.0 / n)
    j1 = orc.JitSpec(11, K, n, orc.LAW_HOMO, 0.6)
    j2 = orc.JitSpec(12, K, n, orc.LAW_HOMO, 0.45)
    ji = orc.JitSpec(13, K, n, orc.LAW_HOMO, 6.7)
    projs = [orc.Projection(0, n1, jit=j1, receptor="exc"),
             orc.Projection(n1, n_exc - n1, jit=j2, receptor="exc"),
             orc.Projection(n_exc, n - n_exc, jit=ji, receptor="inh")]
    st = dict(v=inputs.lif_v0(n), g_e=np.zeros(n, np.int64), g_i=np.zeros(n, np.int64),
              ref=np.zeros(n, np.uint8), spikes=np.zeros(n, np.uint8))
    raster = orc.run_network("lif", orc.lif_params(), st, projs, None, T)
    assert raster.sum() > 0
    dense = []
    for p in projs[:2]:
        d = np.zeros((p.n_rows, n))
        for r in range(p.n_rows):
            d[r, orc.jit_row(p.jit, n, r)[0]] = float(np.float32(p.jit.w0))
        dense.append(d)
    a = math.exp(-0.1 / 5.0)
    g = np.zeros(n)
    prev = np.zeros(n)
    for step in range(T):
        g = a * g + prev[:n1] @ dense[0] + prev[n1:n_exc] @ dense[1]
        prev = raster[step].astype(np.float64)
    g *= a
    assert np.max(np.abs(st["g_e"] / 2.0 ** 32 - g)) < 2.0 ** -20 * max(1.0, g.max())


def test_merged_f32_increment_is_the_exactly_rounded_sum(orc):
    """One neuron receives k1 events of w1 = fl32(0.6) and k2 of w2 =
    fl32(0.45) from two projections into g_E in one step: the increment is
    round_f32(k1 w1 + k2 w2) in exact rationals -- which for some (k1, k2)
    differs from adding the two per-projection roundings."""
    from fractions import Fraction
    w1, w2 = np.float32(0.6), np.float32(0.45)
    differs = 0
    for k1, k2 in ((1, 1), (1, 3), (2, 11), (5, 7), (10, 13), (37, 80), (129, 3), (1000, 999)):
        n = k1 + k2 + 32
        projs = []
        for r0, k, w in ((0, k1, w1), (k1, k2, w2)):
            ip = np.arange(k + 1, dtype=np.int64)       # every row -> column 0
            projs.append(orc.Projection(r0, k, csr=(ip, np.zeros(k, np.int32), None),
                                        w_homo=float(w), receptor="exc"))
        spikes = np.zeros(n, np.uint8)
        spikes[:k1 + k2] = 1
        st = dict(v=np.full(n, -60.0, np.float32), g_e=np.zeros(n, np.float32),
                  g_i=np.zeros(n, np.float32), ref=np.zeros(n, np.uint8), spikes=spikes)
        orc.run_network("lif", orc.lif_params(tau_e=float("inf")), st, projs, None, 1)
        want = _round_f32_exact(k1 * Fraction(float(w1)) + k2 * Fraction(float(w2)))
        assert st["g_e"][0].view(np.uint32) == want.view(np.uint32), (k1, k2)
        two = np.float32(_round_f32_exact(k1 * Fraction(float(w1))) +
                         _round_f32_exact(k2 * Fraction(float(w2))))
        differs += int(two != want)
    assert differs > 0
