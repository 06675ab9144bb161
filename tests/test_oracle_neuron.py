"""Pins for the oracle's neuron/synapse rules N1 (LIF + Expon + COBA) and H1 (HH).

Closed forms: subthreshold exponential decay (exact for the linear ODE of
P:424), the LIF first passage t* = -tau ln(1 - (V_th - V_rest)/(R I)),
the COBA current at E = 0, V = -60, g = 0.6, the Expon decay
g = e^-1 at dt = tau and its semigroup property.  HH (EXTERNAL, not
defined by the paper) is pinned against an independent fp64 RK4 integration
of the same ODEs at dt = 1e-3 ms and by first-order convergence in dt.
"""
import math

import numpy as np
import pytest


def _lif_state(n, v0, fixed=False):
    v = np.full(n, v0, np.float32) if np.isscalar(v0) else np.asarray(v0, np.float32).copy()
    g_dtype = np.int64 if fixed else np.float32
    return v, np.zeros(n, g_dtype), np.zeros(n, g_dtype), np.zeros(n, np.uint8)


def test_subthreshold_decay_closed_form(orc):
    # I = 0, g = 0: V_n = V_rest + (V0 - V_rest) e^{-n dt/tau}
    p = orc.lif_params(i_ext=0.0, v_rest=0.0, v_reset=0.0, v_th=1e9)
    v0 = np.linspace(-15.0, 15.0, 64).astype(np.float32)
    v, ge, gi, ref = _lif_state(64, v0)
    for n in range(1, 1001):
        ev = orc.lif_step(p, v, ge, gi, ref)
        assert not ev.any()
        if n in (1, 10, 100, 1000):
            exact = v0.astype(np.float64) * math.exp(-n * 0.1 / 20.0)
            np.testing.assert_allclose(v, exact, rtol=2e-5, atol=1e-6)


def test_subthreshold_decay_paper_params(orc):
    p = orc.lif_params(i_ext=0.0, v_th=1e9)
    v0 = np.float32(-55.0)
    v, ge, gi, ref = _lif_state(1, v0)
    for _ in range(200):
        orc.lif_step(p, v, ge, gi, ref)
    exact = -60.0 + 5.0 * math.exp(-200 * 0.1 / 20.0)
    assert abs(float(v[0]) - exact) < 2e-3


@pytest.mark.parametrize("fixed", [False, True])
def test_first_passage_and_period(orc, fixed):
    """Unconnected neuron from V_reset with I_ext = 20: first passage
    t* = -20 ln(1 - 10/20) = 13.86 ms -> 139 integration steps, then
    50 refractory steps (tau_ref = 5 ms): period 189 steps."""
    p = orc.lif_params()
    v, ge, gi, ref = _lif_state(3, -60.0, fixed)
    spikes = []
    for step in range(1000):
        if orc.lif_step(p, v, ge, gi, ref)[0]:
            spikes.append(step)
    t_star = -20.0 * math.log(1 - 10.0 / 20.0) / 0.1
    assert spikes[0] == math.ceil(t_star) - 1 == 138
    assert np.all(np.diff(spikes) == 189)


def test_refractory_contract(orc):
    # V above threshold at entry -> spike, reset, silent for exactly 50 steps
    p = orc.lif_params(i_ext=1.0e5)   # crosses V_th in one step
    v, ge, gi, ref = _lif_state(1, -49.0)
    spikes = [s for s in range(300) if orc.lif_step(p, v, ge, gi, ref)[0]]
    assert spikes[0] == 0
    assert np.all(np.diff(spikes) == 51)
    # held at V_reset during the refractory period
    p2 = orc.lif_params(i_ext=1.0e5)
    v, ge, gi, ref = _lif_state(1, -49.0)
    orc.lif_step(p2, v, ge, gi, ref)
    for _ in range(50):
        orc.lif_step(p2, v, ge, gi, ref)
        assert v[0] == np.float32(-60.0)


def test_coba_current(orc):
    """E = 0, V = -60, g = 0.6 -> I = 36; one exponential-Euler step
    then gives V' = -24 - 36 e^{-dt/tau}."""
    p = orc.lif_params(i_ext=0.0, v_th=1e9)
    v, ge, gi, ref = _lif_state(1, -60.0)
    ge[0] = 0.6
    orc.lif_step(p, v, ge, gi, ref)
    assert abs(float(v[0]) - (-24.0 - 36.0 * math.exp(-0.1 / 20.0))) < 2e-5
    # V = E: the COBA term vanishes
    v, ge, gi, ref = _lif_state(1, 0.0)
    ge[0] = 5.0
    p0 = orc.lif_params(i_ext=0.0, v_rest=0.0, v_th=1e9)
    orc.lif_step(p0, v, ge, gi, ref)
    assert v[0] == 0.0
    # inhibition (E_I = -80) pulls V down
    v, ge, gi, ref = _lif_state(1, -60.0)
    gi[0] = 1.0
    orc.lif_step(p, v, ge, gi, ref)
    assert abs(float(v[0]) - (-80.0 + 20.0 * math.exp(-0.1 / 20.0))) < 2e-5


def test_expon_decay_fixed_point(orc):
    # g = 1, tau = 5, dt = 5 -> e^{-1}
    p = orc.lif_params(dt=5.0, tau_e=5.0, tau_i=5.0, i_ext=0.0, v_th=1e9)
    v, ge, gi, ref = _lif_state(1, -60.0, fixed=True)
    ge[0] = 2 ** 32
    orc.lif_step(p, v, ge, gi, ref)
    assert abs(int(ge[0]) - 2 ** 32 * math.exp(-1.0)) <= 0.5
    # semigroup: 100 steps of dt=0.1 equal one decay of 10 ms within rounding
    p = orc.lif_params(i_ext=0.0, v_th=1e9)
    v, ge, gi, ref = _lif_state(1, -60.0, fixed=True)
    ge[0] = 3 * 2 ** 32
    gi[0] = 3 * 2 ** 32
    for _ in range(100):
        orc.lif_step(p, v, ge, gi, ref)
    assert abs(int(ge[0]) - 3 * 2 ** 32 * math.exp(-10.0 / 5.0)) <= 100
    assert abs(int(gi[0]) - 3 * 2 ** 32 * math.exp(-10.0 / 10.0)) <= 100


def test_expon_decay_f32(orc):
    p = orc.lif_params(i_ext=0.0, v_th=1e9)
    v, ge, gi, ref = _lif_state(1, -60.0)
    ge[0] = 1.0
    for _ in range(50):
        orc.lif_step(p, v, ge, gi, ref)
    assert abs(float(ge[0]) - math.exp(-5.0 / 5.0)) < 1e-5


def test_expf_accuracy(orc):
    xs = np.concatenate([np.linspace(-87.0, 88.0, 40001),
                         np.linspace(-1.0, 1.0, 4001)]).astype(np.float32)
    worst = 0.0
    for x in xs:
        got = orc.expf(float(x))
        ref = math.exp(float(x))
        worst = max(worst, abs(got - ref) / float(np.spacing(np.float32(ref))))
    assert worst <= 2.0
    assert orc.expf(0.0) == 1.0


# ---------------------------------------------------------------- HH (H1)

def _hh_rates64(V):
    x = V + 63.0

    def ef(u, k):
        return u / math.expm1(u / k) if abs(u) > 1e-12 else k
    return (0.32 * ef(13 - x, 4), 0.28 * ef(x - 40, 5),
            0.128 * math.exp((17 - x) / 18), 4 / (1 + math.exp((40 - x) / 5)),
            0.032 * ef(15 - x, 5), 0.5 * math.exp((10 - x) / 40))


def _hh_rk4_spikes(i_ext, t_end, dt=1e-3):
    """Independent fp64 RK4 of the COBAHH ODEs (Brette 2007, EXTERNAL)."""
    def f(y):
        V, m, h, n = y
        am, bm, ah, bh, an, bn = _hh_rates64(V)
        dV = (10 * (-60 - V) + 20000 * m ** 3 * h * (50 - V)
              + 6000 * n ** 4 * (-90 - V) + i_ext) / 200.0
        return np.array([dV, am * (1 - m) - bm * m, ah * (1 - h) - bh * h,
                         an * (1 - n) - bn * n])
    y = np.array([-65.0, 0.05, 0.6, 0.32])
    out = []
    for k in range(int(round(t_end / dt))):
        k1 = f(y); k2 = f(y + dt / 2 * k1); k3 = f(y + dt / 2 * k2); k4 = f(y + dt * k3)
        yn = y + dt / 6 * (k1 + 2 * k2 + 2 * k3 + k4)
        if yn[0] >= -20 and y[0] < -20:
            out.append((k + 1) * dt)
        y = yn
    return np.array(out)


def _hh_oracle_spikes(orc, i_ext, t_end, dt):
    p = orc.hh_params(dt=dt, i_ext=i_ext)
    v = np.array([-65.0], np.float32); m = np.array([0.05], np.float32)
    h = np.array([0.6], np.float32); nk = np.array([0.32], np.float32)
    ge = np.zeros(1, np.float32); gi = np.zeros(1, np.float32)
    out = []
    for k in range(int(round(t_end / dt))):
        if orc.hh_step(p, v, m, h, nk, ge, gi)[0]:
            out.append((k + 1) * dt)
    return np.array(out)


def test_hh_against_rk4_and_first_order_convergence(orc):
    rk = _hh_rk4_spikes(400.0, 50.0)
    fine = _hh_oracle_spikes(orc, 400.0, 50.0, 0.01)
    coarse = _hh_oracle_spikes(orc, 400.0, 50.0, 0.1)
    assert len(rk) >= 3 and len(fine) >= 3 and len(coarse) >= 3
    isi_rk = np.diff(rk[:3]).mean()
    err_fine = abs(np.diff(fine[:3]).mean() - isi_rk) / isi_rk
    err_coarse = abs(np.diff(coarse[:3]).mean() - isi_rk) / isi_rk
    assert abs(fine[0] - rk[0]) < 0.15
    assert err_fine < 0.02
    assert err_coarse < 0.15
    assert 4.0 < err_coarse / err_fine < 25.0      # exponential Euler is 1st order


def test_hh_singularities_are_finite_and_continuous(orc):
    p = orc.hh_params(dt=0.1)
    for v_sing in (-50.0, -48.0, -23.0):   # 13-x = 0, 15-x = 0, x-40 = 0
        res = []
        for dv in (-1e-3, 0.0, 1e-3):
            v = np.array([v_sing + dv], np.float32); m = np.array([0.05], np.float32)
            h = np.array([0.6], np.float32); nk = np.array([0.32], np.float32)
            z = np.zeros(1, np.float32)
            orc.hh_step(p, v, m, h, nk, z, z.copy())
            res.append((float(v[0]), float(m[0]), float(nk[0])))
        arr = np.array(res)
        assert np.all(np.isfinite(arr))
        assert np.max(np.abs(arr[0] - arr[1])) < 1e-2
        assert np.max(np.abs(arr[2] - arr[1])) < 1e-2
