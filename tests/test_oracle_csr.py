"""Pins for the oracle's event_csrmv (Listing S1, indices[j]).

event_csrmv reaches a plain result: out = D^T s with D the densified CSR
and s the 0/1 event vector.  Brute force in numpy (exact for small-integer
weights in any summation order) pins it; so do the SPEC examples.
"""
import numpy as np
import pytest

from paper_2311_05106_b200 import inputs


def _dense(indptr, indices, data, w_homo, n_rows, n_cols):
    d = np.zeros((n_rows, n_cols), np.float64)
    for r in range(n_rows):
        for j in range(indptr[r], indptr[r + 1]):
            d[r, indices[j]] += w_homo if data is None else data[j]
    return d


def test_random_instances_match_dense_bruteforce(orc):
    rng = np.random.default_rng(2024)
    for trial in range(500):
        n_rows = int(rng.integers(1, 40))
        n_cols = int(rng.integers(1, 40))
        p = float(rng.choice([0.05, 0.2, 0.6]))
        homo = bool(trial % 2)
        ip, ix, dat = inputs.random_csr(n_rows, n_cols, p, seed=trial,
                                        integer_weights=not homo)
        w_homo = float(rng.integers(-3, 4)) if homo else 0.0
        ev = inputs.spike_pattern(n_rows, float(rng.choice([0.001, 0.01, 0.1, 0.5])),
                                  seed=10_000 + trial)
        d = _dense(ip, ix, dat, w_homo, n_rows, n_cols)
        ref = d.T @ ev.astype(np.float64)
        got = orc.event_csrmv(ip, ix, dat, w_homo, n_rows, n_cols, ev, orc.OUT_F64)
        assert np.array_equal(got, ref)
        got_fix = orc.event_csrmv(ip, ix, dat, w_homo, n_rows, n_cols, ev, orc.OUT_FIX)
        assert np.array_equal(got_fix, (ref * 2.0 ** 32).astype(np.int64))
        got32 = orc.event_csrmv(ip, ix, dat, w_homo, n_rows, n_cols, ev, orc.OUT_F32)
        assert np.array_equal(got32.astype(np.float64), ref)


def test_spec_identity_example(orc):
    # S:52 analogue for events: CSR of the 3x3 identity, w = 2.5,
    # events [1, 0, 1] -> [2.5, 0, 2.5].
    ip = np.array([0, 1, 2, 3], np.int64)
    ix = np.array([0, 1, 2], np.int32)
    out = orc.event_csrmv(ip, ix, None, 2.5, 3, 3, np.array([1, 0, 1], np.uint8))
    assert out.tolist() == [2.5, 0.0, 2.5]


def test_all_false_and_single_event(orc):
    ip, ix, dat = inputs.random_csr(30, 50, 0.2, seed=1, weights="uniform",
                                    w0=-1.0, w1=1.0)
    d = _dense(ip, ix, dat, 0.0, 30, 50)
    assert not orc.event_csrmv(ip, ix, dat, 0.0, 30, 50, np.zeros(30, np.uint8)).any()
    for k in (0, 7, 29):
        ev = np.zeros(30, np.uint8)
        ev[k] = 1
        got = orc.event_csrmv(ip, ix, dat, 0.0, 30, 50, ev)
        assert np.array_equal(got, d[k])


def test_fixed_point_quantisation(orc):
    # rule F1: q(w) = round-half-even(w * 2^32)
    for w in [0.6, 6.7, -0.1, 1.0, 0.0, 1e-9, 3.0e-10]:
        w32 = np.float32(w)
        exact = float(w32) * 2.0 ** 32           # exact in fp64
        fl = np.floor(exact)
        frac = exact - fl
        want = fl + (1 if frac > 0.5 or (frac == 0.5 and fl % 2 == 1) else 0)
        assert orc.quantize(float(w32)) == int(want)
    assert orc.quantize(0.5 * 2.0 ** -32) == 0      # tie -> even (0)
    assert orc.quantize(1.5 * 2.0 ** -32) == 2      # tie -> even (2)


def test_fixed_vs_f64_error_bound(orc):
    ip, ix, dat = inputs.random_csr(200, 300, 0.1, seed=4, weights="normal",
                                    w0=0.0, w1=1.0)
    ev = inputs.spike_pattern(200, 0.3, 9)
    f64, absd = orc.event_csrmv(ip, ix, dat, 0.0, 200, 300, ev, orc.OUT_F64,
                                with_abs=True)
    fix = orc.event_csrmv(ip, ix, dat, 0.0, 200, 300, ev, orc.OUT_FIX)
    terms = orc.event_csrmv(ip, ix, None, 1.0, 200, 300, ev, orc.OUT_F64)
    # each term rounds by <= 2^-33; the fp64 sum is exact to ~1e-16 |w|
    err = np.abs(fix / 2.0 ** 32 - f64)
    assert np.all(err <= terms * 2.0 ** -33 + 1e-12 * absd)


@pytest.mark.parametrize("n_rows,n_cols", [(0, 5), (5, 1)])
def test_degenerate_shapes(orc, n_rows, n_cols):
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.5, seed=3)
    ev = np.ones(n_rows, np.uint8)
    out = orc.event_csrmv(ip, ix, dat, 1.0, n_rows, n_cols, ev)
    assert out.shape == (n_cols,)
    d = _dense(ip, ix, dat, 1.0, n_rows, n_cols)
    assert np.array_equal(out, d.sum(axis=0))


# ---------------------------------------------------------------- reading G1
@pytest.mark.parametrize("homo", [True, False])
def test_gather_equals_scatter_of_transpose(orc, homo):
    """Gather orientation on M equals the Listing-S1 scatter on M^T."""
    n_rows, n_cols = 60, 45
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.2, seed=3, integer_weights=not homo)
    w = 0.75
    d = _dense(ip, ix, dat, w, n_rows, n_cols)             # M[r, c]
    # transpose as CSR (rows = columns of M)
    rows_t, cols_t = np.nonzero(d.T)
    ipt = np.zeros(n_cols + 1, np.int64)
    np.add.at(ipt, rows_t + 1, 1)
    ipt = np.cumsum(ipt)
    datt = d.T[rows_t, cols_t].astype(np.float32)
    ev = inputs.spike_pattern(n_cols, 0.4, 8)
    got = orc.csrmv_gather(ip, ix, dat, w, n_rows, n_cols, ev, out_kind=orc.OUT_FIX)
    want = orc.event_csrmv(ipt, cols_t.astype(np.int32), datt, 0.0, n_cols, n_rows, ev,
                           orc.OUT_FIX)
    assert np.array_equal(got, want)
    assert np.allclose(orc.csrmv_gather(ip, ix, dat, w, n_rows, n_cols, ev), d @ ev)


@pytest.mark.parametrize("homo", [True, False])
def test_grad_matches_torch_autograd(orc, homo):
    """dL/ddata, dL/ds and dL/dw of L = gy . (M^T s) against torch autograd
    of the dense fp64 product (an independent computation)."""
    import torch
    n_rows, n_cols = 50, 70
    ip, ix, dat = inputs.random_csr(n_rows, n_cols, 0.15, seed=5,
                                    weights="homo" if homo else "uniform", w0=-1.0, w1=1.0)
    w = float(np.float32(0.6))                  # the oracle's weights are fp32
    ev = inputs.spike_pattern(n_rows, 0.5, 2)
    rng = np.random.default_rng(4)
    gy = rng.normal(size=n_cols).astype(np.float32)
    rows = np.repeat(np.arange(n_rows), np.diff(ip))
    vals = torch.tensor(np.full(ix.shape[0], w) if homo else dat.astype(np.float64),
                        requires_grad=True)
    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    s = torch.tensor(ev.astype(np.float64), requires_grad=True)
    dense = torch.zeros(n_rows, n_cols, dtype=torch.float64)
    dense = dense.index_put((torch.tensor(rows), torch.tensor(ix.astype(np.int64))),
                            vals * (wt / w if homo else 1.0), accumulate=True)
    y = dense.T @ s
    (y @ torch.tensor(gy.astype(np.float64))).backward()
    gd, ge, gw = orc.csrmv_grad(ip, ix, None if homo else dat, w, n_rows, ev, gy)
    assert np.allclose(ge, s.grad.numpy(), rtol=1e-12, atol=1e-12)
    if homo:
        assert abs(gw - wt.grad.item()) <= 1e-9 * max(1.0, abs(gw))
    else:
        assert np.allclose(gd.astype(np.float64), vals.grad.numpy(), rtol=0, atol=0)
