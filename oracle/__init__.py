"""CPU oracle for the BrainPy hot path -- TEST INFRASTRUCTURE ONLY.

Thin numpy/ctypes wrapper around ``liboracle.so`` (built from
``oracle/bp_oracle.c``) plus the network time loop of rule S1 written out in
Python.  Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package; the
product package ``paper_2311_05106_b200`` never does, and the two share no
code.

Spike vectors here are plain ``uint8`` arrays, one entry per neuron, exactly
the ``events`` of Listing S1/S2.  Conversion from the
product's bit-packed words is done by the tests, not here.

Parity status per function:
  philox / conn_len / jit_row / jit_event_mv / event_csrmv /
  lif_step / hh_step / expf / run_network: pinned (tests/test_oracle_*.py);
  run_network's fp32 conductance branch (rule N1-f32, the bench's default
  mode) by the exactly rounded increment (exact rational arithmetic) and the
  fp64 recursion within its rounding bound (test_oracle_network.py).
  run_network firing *rates*: parity unpinned by the paper (reading R23) --
  the paper prints no COBA statistics; rasters are pinned only through the
  closed-form w = 0 network and the per-step primitives.
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "bp_oracle.c")
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OUT_F64, OUT_FIX, OUT_F32, OUT_FIX32 = 0, 1, 2, 3
LAW_HOMO, LAW_UNIFORM, LAW_NORMAL = 0, 1, 2
LAWS = {"homo": LAW_HOMO, "uniform": LAW_UNIFORM, "normal": LAW_NORMAL}

BUILD_CMD = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math",
             "-fopenmp", "-fPIC", "-shared", "-o", _LIB_PATH, _SRC, "-lm"]


def build() -> str:
    """Compile liboracle.so (gcc, -ffp-contract=off) if it is missing or stale."""
    if (not os.path.exists(_LIB_PATH)
            or os.path.getmtime(_LIB_PATH) < os.path.getmtime(_SRC)):
        subprocess.check_call(BUILD_CMD)
    return _LIB_PATH


class LifParams(ctypes.Structure):
    _fields_ = [("v_rest", ctypes.c_float), ("v_reset", ctypes.c_float),
                ("v_th", ctypes.c_float), ("r", ctypes.c_float),
                ("i_ext", ctypes.c_float), ("e_exc", ctypes.c_float),
                ("e_inh", ctypes.c_float), ("alpha_v", ctypes.c_float),
                ("alpha_e", ctypes.c_double), ("alpha_i", ctypes.c_double),
                ("ref_steps", ctypes.c_int32), ("pad_", ctypes.c_int32)]


class HHParams(ctypes.Structure):
    _fields_ = [(name, ctypes.c_float) for name in
                ("c_m", "g_l", "e_l", "g_na", "e_na", "g_k", "e_k", "v_t",
                 "e_exc", "e_inh", "i_ext", "dt", "v_spike", "pad_")] + \
               [("alpha_e", ctypes.c_double), ("alpha_i", ctypes.c_double)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        u32, u64, i64, f32, f64, i32 = (ctypes.c_uint32, ctypes.c_uint64,
                                        ctypes.c_int64, ctypes.c_float,
                                        ctypes.c_double, ctypes.c_int)
        _lib.or_philox4x32_10.argtypes = [P, P, P]
        _lib.or_word.argtypes = [u64, u32, u32, u32, u32]
        _lib.or_word.restype = u32
        _lib.or_conn_len.argtypes = [f64]
        _lib.or_conn_len.restype = u32
        _lib.or_quantize.argtypes = [f32]
        _lib.or_quantize.restype = i64
        _lib.or_jit_row.argtypes = [u64, u32, u32, i64, i32, f32, f32, u32,
                                    i64, i64, P, P, i64]
        _lib.or_jit_row.restype = i64
        _lib.or_event_csrmv.argtypes = [P, P, P, f32, i64, P, i32, P, P]
        _lib.or_jit_event_mv.argtypes = [u64, u32, u32, i32, f32, f32, i64,
                                         i64, i64, i64, P, i32, P, P]
        _lib.or_csrmv_gather.argtypes = [P, P, P, f32, i64, P, i32, P, P]
        _lib.or_csrmv_grad.argtypes = [P, P, P, f32, i64, P, P, P, P, P]
        _lib.or_jit_mv.argtypes = [u64, u32, u32, i32, f32, f32, i64, i64, i64, i64,
                                   P, i32, P, P]
        _lib.or_lif_step.argtypes = [ctypes.POINTER(LifParams), i64, P, P, P,
                                     i32, P, P]
        _lib.or_hh_step.argtypes = [ctypes.POINTER(HHParams), i64, P, P, P, P,
                                    P, P, i32, P]
        _lib.or_expf.argtypes = [f32]
        _lib.or_expf.restype = f32
        _lib.or_set_fix32_bits.argtypes = [i32]
        _lib.or_set_gap_sampler.argtypes = [f32]
        _lib.or_geo_c.argtypes = [f64]
        _lib.or_geo_c.restype = f32
        _lib.or_logf_j10.argtypes = [f32]
        _lib.or_logf_j10.restype = f32
        _lib.or_cos2pi_j7.argtypes = [f32]
        _lib.or_cos2pi_j7.restype = f32
        _lib.or_gap_draws.argtypes = [i32, f64, u64, u64]
        _lib.or_gap_draws.restype = u64
        _lib.or_geo_gap.argtypes = [f32, u32, u32]
        _lib.or_geo_gap.restype = u32
        _lib.or_fix32_add.argtypes = [P, P, i64]
        _lib.or_fix32_add.restype = i64
        _lib.or_set_threads.argtypes = [i32]
        _lib.or_get_threads.restype = i32
    return _lib


def _p(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


# --------------------------------------------------------------------------
# RNG and connectivity rules (J1-J7)
# --------------------------------------------------------------------------

def philox(ctr, key) -> np.ndarray:
    c = np.asarray(ctr, dtype=np.uint32)
    k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c), _p(k), _p(out))
    return out


def word(seed: int, tag: int, row: int, seg: int, j: int) -> int:
    return int(lib().or_word(seed, tag, row, seg, j))


def conn_len(p: float) -> int:
    return int(lib().or_conn_len(float(p)))


def quantize(w: float) -> int:
    return int(lib().or_quantize(float(w)))


def expf(x: float) -> float:
    return float(lib().or_expf(float(x)))


@dataclass(frozen=True)
class JitSpec:
    """Rule J-spec: (seed, K, L) fix the matrix; (law, w0, w1) the weights."""
    seed: int
    K: int
    L: int  # seg_len; the segment grid is part of the connectivity (rule J4)
    law: int = LAW_HOMO
    w0: float = 1.0
    w1: float = 0.0
    # rule J10: 0 -> uniform gaps U[1, K] (J3); else c = fl32(log1p(-p)) and
    # gaps are Geo(p) by inversion (geometric sampler)
    geo_c: float = 0.0


def geo_c(p: float) -> float:
    """Rule J10 constant c = fl32(log1p(-p))."""
    return float(lib().or_geo_c(p))


def logf_j10(u: float) -> float:
    """Rule J10's specified fp32 natural log."""
    return float(lib().or_logf_j10(u))


def cos2pi_j7(u: float) -> float:
    """Reading J7n's specified fp32 cos(2 pi u)."""
    return float(lib().or_cos2pi_j7(u))


def gap_draws(geometric: bool, p: float, n: int, seed: int = 1) -> int:
    """Sum of n gap draws (sampler-cost probe): U[1, K] or Geo(p)."""
    return int(lib().or_gap_draws(1 if geometric else 0, p, n, seed))


def geo_gap(c: float, cap: int, x: int) -> int:
    """Rule J10 gap from one 32-bit word x."""
    return int(lib().or_geo_gap(c, cap, x))


class _Sampler:
    """Selects the gap sampler of one oracle call (rule J3 or J10)."""

    def __init__(self, spec):
        self.c = spec.geo_c

    def __enter__(self):
        lib().or_set_gap_sampler(self.c)

    def __exit__(self, *exc):
        lib().or_set_gap_sampler(0.0)


def jit_row(spec: JitSpec, n_cols: int, row: int, seg_first: int = 0,
            seg_last: int | None = None):
    """(positions int32, weights float32) of one row, segments seg_first..seg_last."""
    if seg_last is None:
        seg_last = (n_cols - 1) // spec.L
    cap = 64
    while True:
        pos = np.empty(cap, np.int32)
        w = np.empty(cap, np.float32)
        with _Sampler(spec):
            n = lib().or_jit_row(spec.seed, spec.K, spec.L, n_cols, spec.law,
                                 spec.w0, spec.w1, row, seg_first, seg_last,
                                 _p(pos), _p(w), cap)
        if n <= cap:
            return pos[:n].copy(), w[:n].copy()
        cap = int(n)


def jit_materialize(spec: JitSpec, n_rows: int, n_cols: int):
    """CSR (indptr int64, indices int32, data float32) of the implied matrix."""
    rows = [jit_row(spec, n_cols, r) for r in range(n_rows)]
    indptr = np.zeros(n_rows + 1, np.int64)
    indptr[1:] = np.cumsum([len(p) for p, _ in rows])
    indices = (np.concatenate([p for p, _ in rows]) if n_rows else
               np.zeros(0, np.int32)).astype(np.int32)
    data = (np.concatenate([w for _, w in rows]) if n_rows else
            np.zeros(0, np.float32)).astype(np.float32)
    return indptr, indices, data


def _out_buf(n: int, out_kind: int):
    return np.zeros(n, {OUT_F64: np.float64, OUT_FIX: np.int64,
                        OUT_F32: np.float32, OUT_FIX32: np.int64}[out_kind])


def set_threads(n: int):
    """Host threads for the order-free loops (per-neuron updates, integer
    event scatters); results are bit-identical to 1 thread (see the C
    header).  Test-time speed only."""
    lib().or_set_threads(int(n))


def get_threads() -> int:
    return int(lib().or_get_threads())


def set_fix32_bits(bits: int):
    """Rule F2: fractional bits of the 32-bit fixed-point conductances."""
    lib().or_set_fix32_bits(int(bits))


def fix32_add(g: np.ndarray, inc: np.ndarray) -> int:
    """Rule F2: g (int32) += inc (int64, exact step sum) with saturation."""
    assert g.dtype == np.int32 and inc.dtype == np.int64
    return int(lib().or_fix32_add(_p(g), _p(inc), g.shape[0]))


def event_csrmv(indptr, indices, data, w_homo, n_rows, n_cols, events,
                out_kind=OUT_F64, out=None, with_abs=False):
    """Listing S1 (indices[j] reading). Returns out (and sum|w| if with_abs)."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    data = None if data is None else np.ascontiguousarray(data, np.float32)
    ev = np.ascontiguousarray(events, np.uint8)
    assert ev.shape[0] == n_rows
    if out is None:
        out = _out_buf(n_cols, out_kind)
    absd = np.zeros(n_cols, np.float64) if with_abs else None
    lib().or_event_csrmv(_p(indptr), _p(indices), _p(data), float(w_homo),
                         n_rows, _p(ev), out_kind, _p(out), _p(absd))
    return (out, absd) if with_abs else out


def csrmv_gather(indptr, indices, data, w_homo, n_rows, n_cols, events,
                 out_kind=OUT_F64, out=None, with_abs=False):
    """Gather orientation (transpose=False, reading G1): out[r] = sum over
    row r of w_k [events[indices[k]]]; events has n_cols entries."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    data = None if data is None else np.ascontiguousarray(data, np.float32)
    ev = np.ascontiguousarray(events, np.uint8)
    assert ev.shape[0] == n_cols
    if out is None:
        out = _out_buf(n_rows, out_kind)
    absd = np.zeros(n_rows, np.float64) if with_abs else None
    lib().or_csrmv_gather(_p(indptr), _p(indices), _p(data), float(w_homo), n_rows, _p(ev),
                          out_kind, _p(out), _p(absd))
    return (out, absd) if with_abs else out


def csrmv_grad(indptr, indices, data, w_homo, n_rows, events, gy):
    """Reverse mode of the event scatter y = M^T s (reading G1): returns
    (grad_data f32[nnz], grad_events f64[n_rows], grad_w f64)."""
    indptr = np.ascontiguousarray(indptr, np.int64)
    indices = np.ascontiguousarray(indices, np.int32)
    data = None if data is None else np.ascontiguousarray(data, np.float32)
    ev = np.ascontiguousarray(events, np.uint8)
    gy = np.ascontiguousarray(gy, np.float32)
    gd = np.zeros(indices.shape[0], np.float32)
    ge = np.zeros(n_rows, np.float64)
    gw = np.zeros(1, np.float64)
    lib().or_csrmv_grad(_p(indptr), _p(indices), _p(data), float(w_homo), n_rows, _p(ev),
                        _p(gy), _p(gd), _p(ge), _p(gw))
    return gd, ge, float(gw[0])


def jit_event_mv(spec: JitSpec, n_rows, n_cols, events, col_begin=0,
                 col_end=None, out_kind=OUT_F64, out=None, with_abs=False):
    """Listing S2 / rule J9 over columns [col_begin, col_end)."""
    if col_end is None:
        col_end = n_cols
    ev = np.ascontiguousarray(events, np.uint8)
    assert ev.shape[0] == n_rows
    if out is None:
        out = _out_buf(col_end - col_begin, out_kind)
    absd = np.zeros(col_end - col_begin, np.float64) if with_abs else None
    with _Sampler(spec):
        lib().or_jit_event_mv(spec.seed, spec.K, spec.L, spec.law, spec.w0,
                              spec.w1, n_rows, n_cols, col_begin, col_end,
                              _p(ev), out_kind, _p(out), _p(absd))
    return (out, absd) if with_abs else out


def jit_mv(spec: JitSpec, n_rows, n_cols, v, col_begin=0, col_end=None,
           out_kind=OUT_F64, out=None, with_abs=False):
    """Non-event mv_prob_* (reading MV1): out[c] += sum_r v[r] w_e."""
    if col_end is None:
        col_end = n_cols
    vv = np.ascontiguousarray(v, np.float32)
    assert vv.shape[0] == n_rows
    if out is None:
        out = _out_buf(col_end - col_begin, out_kind)
    absd = np.zeros(col_end - col_begin, np.float64) if with_abs else None
    with _Sampler(spec):
        lib().or_jit_mv(spec.seed, spec.K, spec.L, spec.law, spec.w0, spec.w1, n_rows,
                        n_cols, col_begin, col_end, _p(vv), out_kind, _p(out), _p(absd))
    return (out, absd) if with_abs else out


# --------------------------------------------------------------------------
# Neuron rules N1 / H1
# --------------------------------------------------------------------------

def lif_params(dt=0.1, tau=20.0, tau_e=5.0, tau_i=10.0, v_rest=-60.0,
               v_reset=-60.0, v_th=-50.0, r=1.0, i_ext=20.0, e_exc=0.0,
               e_inh=-80.0, tau_ref=5.0) -> LifParams:
    """Listing S3 constants; alphas evaluated once, fp64."""
    return LifParams(v_rest, v_reset, v_th, r, i_ext, e_exc, e_inh,
                     np.float32(math.exp(-dt / tau)), math.exp(-dt / tau_e),
                     math.exp(-dt / tau_i), int(round(tau_ref / dt)), 0)


def hh_params(dt=0.1, tau_e=5.0, tau_i=10.0, i_ext=0.0) -> HHParams:
    """Rule H1 constants (Brette et al. 2007 COBAHH; EXTERNAL)."""
    return HHParams(200.0, 10.0, -60.0, 20000.0, 50.0, 6000.0, -90.0, -63.0,
                    0.0, -80.0, i_ext, dt, -20.0, 0.0,
                    math.exp(-dt / tau_e), math.exp(-dt / tau_i))


def lif_step(params: LifParams, v, g_e, g_i, ref):
    """In-place rule N1 on numpy arrays; returns the uint8 spike vector."""
    n = v.shape[0]
    g_kind = {np.dtype(np.int64): 1, np.dtype(np.int32): 2}.get(g_e.dtype, 0)
    ev = np.zeros(n, np.uint8)
    lib().or_lif_step(ctypes.byref(params), n, _p(v), _p(g_e), _p(g_i),
                      g_kind, _p(ref), _p(ev))
    return ev


def hh_step(params: HHParams, v, m, h, nk, g_e, g_i):
    n = v.shape[0]
    g_kind = {np.dtype(np.int64): 1, np.dtype(np.int32): 2}.get(g_e.dtype, 0)
    ev = np.zeros(n, np.uint8)
    lib().or_hh_step(ctypes.byref(params), n, _p(v), _p(m), _p(h), _p(nk),
                     _p(g_e), _p(g_i), g_kind, _p(ev))
    return ev


# --------------------------------------------------------------------------
# Rule S1: the network time loop (Listing S3 update())
# --------------------------------------------------------------------------

@dataclass
class Projection:
    """Rows = presynaptic neurons [row0, row0 + n_rows); cols = all N posts.
    receptor: 'exc' (adds into g_e) or 'inh' (g_i); None = by position in
    run_network's (proj_e, proj_i) pair."""
    row0: int
    n_rows: int
    jit: JitSpec | None = None
    csr: tuple | None = None        # (indptr, indices, data or None)
    w_homo: float = 0.0             # CSR homogeneous weight when data is None
    receptor: str | None = None

    @property
    def weight(self) -> float:
        return float(self.jit.w0) if self.jit is not None else float(self.w_homo)

    @property
    def homogeneous(self) -> bool:
        return (self.jit is not None and self.jit.law == LAW_HOMO
                or self.jit is None and self.csr[2] is None)


def _counts(proj: Projection, ev, n_total, col_begin, col_end, out):
    """Number of events of `proj` per postsynaptic column (Listing S1 / S2
    with unit weights; exact integers in fp64), accumulated into out."""
    if proj.jit is not None:
        spec1 = JitSpec(proj.jit.seed, proj.jit.K, proj.jit.L, LAW_HOMO, 1.0,
                        geo_c=proj.jit.geo_c)
        jit_event_mv(spec1, proj.n_rows, n_total, ev, col_begin, col_end, OUT_F64, out=out)
    else:
        ip, ix, _ = proj.csr
        event_csrmv(ip, ix, None, 1.0, proj.n_rows, col_end - col_begin, ev, OUT_F64, out=out)


def _f32_increment(projs, spikes, n_total, col_begin, col_end, n_local):
    """Rule N1-f32 for the homogeneous projections of one receptor: the
    step's increment is the EXACTLY ROUNDED sum of its events' weights,
    fl32(sum_p count_p w_p) (AlignPost merging: one conductance for
    all of them).  Projections with equal weights are counted together; one
    weight: fl32(count w) (count w is exact in fp64); several: the exact sum
    in integer units of 2^-32 (every weight must be a multiple of 2^-32),
    rounded once to fp32.  Returns (nonzero mask, fp32 increment)."""
    groups = {}
    for proj in projs:
        w = np.float32(proj.weight)
        cnt = groups.setdefault(w.tobytes(), (w, np.zeros(n_local, np.float64)))[1]
        ev = spikes[proj.row0:proj.row0 + proj.n_rows]
        _counts(proj, ev, n_total, col_begin, col_end, cnt)
    if len(groups) == 1:
        (w, cnt), = groups.values()
        return cnt != 0, (cnt.astype(np.float32) * w).astype(np.float32)
    S = np.zeros(n_local, np.int64)
    for w, cnt in groups.values():
        q = float(w) * 4294967296.0
        assert q == math.floor(q), "merged fp32 weights must lie on the 2^-32 grid"
        S += cnt.astype(np.int64) * np.int64(q)
    return S != 0, (S.astype(np.float32) * np.float32(2.0 ** -32)).astype(np.float32)


def run_network(model: str, params, state: dict, proj_e: Projection,
                proj_i: Projection | None, n_steps: int, col_begin: int = 0,
                col_end: int | None = None, record=True, delay: int = 1):
    """Rule S1, for n = 0 .. n_steps-1:
        1. read spikes_{n-D} (D = delay steps, reading D1; D = 1 is the
           paper's one-step VarDelay, P:971/P:988/P:991)
        2. every projection adds its events into the conductance of its
           receptor (E rows -> g_E, I rows -> g_I in Listing S3; a2/a4);
           projections of one receptor merge into its single g
        3. neuron rule N1 (LIF) or H1 (HH) -> spikes_n
        4. store spikes_n
    proj_e, proj_i: Listing S3's two projections; or proj_e = a LIST of
    projections (each with .receptor) and proj_i = None.
    `state` holds numpy arrays (v, g_e, g_i, ref | m, h, n) over the
    postsynaptic columns [col_begin, col_end) and 'spikes' (uint8, all N):
    spikes_{-1} on entry (spikes_{-2}, ..., spikes_{-D} are empty unless
    state['history'] holds them, oldest first), spikes_{n_steps-1} on exit.
    g dtype int64 selects fixed point (rule F1), int32 rule F2, float32 fp32.
    Returns the raster (n_steps x N uint8) when record, else spike counts.
    """
    assert delay >= 1
    if isinstance(proj_e, (list, tuple)):
        projs = list(proj_e)
    else:
        projs = [proj_e, proj_i]
        for p, r in zip(projs, ("exc", "inh")):
            if p.receptor is None:
                p.receptor = r
    by_rec = {"exc": [p for p in projs if p.receptor == "exc"],
              "inh": [p for p in projs if p.receptor == "inh"]}
    assert len(by_rec["exc"]) + len(by_rec["inh"]) == len(projs)
    hist = state.get("history")
    if delay == 1 or hist is None or len(hist) != delay:
        hist = [np.zeros_like(state["spikes"]) for _ in range(delay - 1)] + [state["spikes"]]
    n_total = state["spikes"].shape[0]
    if col_end is None:
        col_end = n_total
    n_local = col_end - col_begin
    fix32 = state["g_e"].dtype == np.int32
    fixed = state["g_e"].dtype == np.int64
    f32 = not (fix32 or fixed)
    kind = OUT_FIX32 if fix32 else (OUT_FIX if fixed else OUT_F32)
    raster = np.zeros((n_steps, n_local), np.uint8) if record else None
    counts = np.zeros(n_steps, np.int64)
    for step in range(n_steps):
        spikes = hist[0]
        for rec, g in (("exc", state["g_e"]), ("inh", state["g_i"])):
            group = by_rec[rec]
            if not group:
                continue
            if f32 and all(p.homogeneous for p in group):
                nz, inc = _f32_increment(group, spikes, n_total, col_begin, col_end, n_local)
                g[nz] = g[nz] + inc[nz]
                continue
            # fixed point: the increments of every projection of the receptor
            # summed exactly (int64) -- rule F1 adds them straight into g,
            # rule F2 adds the step's sum to the int32 g with saturation;
            # fp32 with heterogeneous weights: sequential fp32 accumulation
            acc = np.zeros(n_local, np.int64) if fix32 else g
            for proj in group:
                ev = spikes[proj.row0:proj.row0 + proj.n_rows]
                if proj.jit is not None:
                    jit_event_mv(proj.jit, proj.n_rows, n_total, ev, col_begin,
                                 col_end, kind, out=acc)
                else:
                    ip, ix, dat = proj.csr
                    event_csrmv(ip, ix, dat, proj.w_homo, proj.n_rows,
                                n_local, ev, kind, out=acc)
            if fix32:
                fix32_add(g, acc)
        if model == "lif":
            local = lif_step(params, state["v"], state["g_e"], state["g_i"],
                             state["ref"])
        else:
            local = hh_step(params, state["v"], state["m"], state["h"],
                            state["n"], state["g_e"], state["g_i"])
        new = np.zeros(n_total, np.uint8)
        new[col_begin:col_end] = local
        state["spikes"] = new
        hist = hist[1:] + [new]
        counts[step] = int(local.sum())
        if record:
            raster[step] = local
    state["history"] = hist
    return raster if record else counts
