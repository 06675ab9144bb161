"""ctypes binding of libbp.so (include/bp.h) -- argument marshalling only.

Every function takes torch tensors that live on the current CUDA device and
passes their data pointers, sizes and the current stream to the C ABI; all
computation happens in the library's sm_100a kernels.  There is no CPU
fallback: if libbp.so is missing or the device is not sm_100, calls raise.
"""
from __future__ import annotations

import ctypes
import math
import os

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# BP_LIB overrides the library path (A/B experiments with alternative builds)
LIB_PATH = os.environ.get("BP_LIB") or os.path.join(_HERE, "libbp.so")

OUT_F32, OUT_FIX64, OUT_FIX32 = 0, 1, 2
ACCUMULATE = 1
LAW_HOMO, LAW_UNIFORM, LAW_NORMAL = 0, 1, 2
MODEL_LIF, MODEL_HH = 0, 1
CONN_JIT, CONN_CSR = 0, 1

EXPORTED = [
    "bp_abi_version", "bp_status_string", "bp_last_error", "bp_conn_len",
    "bp_workspace_bytes", "bp_csrmv_workspace_bytes", "bp_compact_spikes", "bp_event_csrmv",
    "bp_csrmv_plan_bytes", "bp_csrmv_plan", "bp_event_csrmv_planned",
    "bp_jitconn_workspace_bytes", "bp_jitconn_mv_homo", "bp_jitconn_mv_uniform",
    "bp_jitconn_mv_normal", "bp_csrmv_gather", "bp_event_csrmv_grad",
    "bp_jitconn_event_mv_homo", "bp_jitconn_event_mv_uniform",
    "bp_jitconn_event_mv_normal", "bp_jitconn_row_counts", "bp_jitconn_indptr",
    "bp_jitconn_materialize", "bp_neuron_step", "bp_network_workspace_bytes",
    "bp_network_create", "bp_network_step", "bp_network_scatter",
    "bp_network_update", "bp_network_update_overlap", "bp_network_counters", "bp_network_profile_begin",
    "bp_network_profile_end", "bp_network_destroy", "bp_network_device_bytes",
    "bp_nccl_unique_id", "bp_network_describe", "bp_nccl_version",
]


class BpError(RuntimeError):
    pass


class JitConn(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("prob", ctypes.c_double),
                ("conn_len", ctypes.c_uint32), ("seg_len", ctypes.c_uint32),
                ("gap_law", ctypes.c_int32), ("reserved", ctypes.c_int32)]


GAP_UNIFORM, GAP_GEOMETRIC = 0, 1   # bp_gap_law (include/bp.h)


_F = ctypes.c_float


class NeuronParams(ctypes.Structure):
    _fields_ = ([("model", ctypes.c_int32), ("ref_steps", ctypes.c_int32)] +
                [(n, _F) for n in ("v_rest", "v_reset", "v_th", "r", "i_ext",
                                   "e_exc", "e_inh", "alpha_v")] +
                [("alpha_e", ctypes.c_double), ("alpha_i", ctypes.c_double)] +
                [(n, _F) for n in ("c_m", "g_l", "e_l", "g_na", "e_na", "g_k",
                                   "e_k", "v_t", "dt", "v_spike")])


class NeuronState(ctypes.Structure):
    _fields_ = [("v", ctypes.c_void_p), ("g_exc", ctypes.c_void_p),
                ("g_inh", ctypes.c_void_p), ("g_kind", ctypes.c_int32),
                ("g_frac_bits", ctypes.c_int32), ("ref", ctypes.c_void_p),
                ("m", ctypes.c_void_p), ("h", ctypes.c_void_p),
                ("n_gate", ctypes.c_void_p)]


class CsrmvPlanInfo(ctypes.Structure):
    _fields_ = [("n_tiles", ctypes.c_int32), ("f32_fixed_bits", ctypes.c_int32),
                ("max_col_abs_sum", ctypes.c_double)]


MAX_PROJ = 8                            # BP_MAX_PROJ
RECEPTOR_EXC, RECEPTOR_INH = 0, 1
EXCHANGE_CALLER, EXCHANGE_NCCL = 0, 1


class Projection(ctypes.Structure):
    _fields_ = [("conn", ctypes.c_int32), ("receptor", ctypes.c_int32),
                ("pre_begin", ctypes.c_int64), ("pre_end", ctypes.c_int64),
                ("weight", _F), ("reserved", ctypes.c_int32), ("jit", JitConn),
                ("indptr", ctypes.c_void_p), ("indices", ctypes.c_void_p)]


class NetworkDesc(ctypes.Structure):
    _fields_ = [("model", ctypes.c_int32), ("g_kind", ctypes.c_int32),
                ("delay_steps", ctypes.c_int32), ("n_proj", ctypes.c_int32),
                ("n", ctypes.c_int64),
                ("col_begin", ctypes.c_int64), ("col_end", ctypes.c_int64),
                ("proj", Projection * MAX_PROJ),
                ("params", NeuronParams), ("state", NeuronState),
                ("spikes", ctypes.c_void_p), ("ws", ctypes.c_void_p),
                ("ws_bytes", ctypes.c_size_t),
                ("exchange", ctypes.c_int32), ("rank", ctypes.c_int32),
                ("world", ctypes.c_int32), ("reserved2", ctypes.c_int32),
                ("part_len", ctypes.c_int64), ("nccl_id", ctypes.c_uint8 * 128)]


_lib = None


def lib():
    """Load libbp.so; raise loudly if it was not built (no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise BpError(f"{LIB_PATH} not built: run __graft_entry__.build()")
        L = ctypes.CDLL(LIB_PATH)
        P, i64, u32, f32, i32 = (ctypes.c_void_p, ctypes.c_int64,
                                 ctypes.c_uint32, ctypes.c_float, ctypes.c_int)
        sz = ctypes.c_size_t
        L.bp_status_string.restype = ctypes.c_char_p
        L.bp_last_error.restype = ctypes.c_char_p
        L.bp_conn_len.argtypes = [ctypes.c_double]
        L.bp_conn_len.restype = u32
        L.bp_workspace_bytes.argtypes = [i64]
        L.bp_workspace_bytes.restype = sz
        L.bp_csrmv_workspace_bytes.argtypes = [i64, i64, i32]
        L.bp_csrmv_workspace_bytes.restype = sz
        L.bp_compact_spikes.argtypes = [P, i64, P, P, P]
        L.bp_event_csrmv.argtypes = [P, P, P, f32, i64, i64, P, P, i32, u32, P, sz, P]
        L.bp_jitconn_workspace_bytes.argtypes = [i64, i64, i64, i32]
        L.bp_jitconn_workspace_bytes.restype = sz
        L.bp_csrmv_gather.argtypes = [P, P, P, f32, i64, i64, P, P, i32, u32, P]
        L.bp_event_csrmv_grad.argtypes = [P, P, P, f32, i64, i64, P, P, P, P, P, P]
        L.bp_csrmv_plan_bytes.argtypes = [i64, i64, i32, i32]
        L.bp_csrmv_plan_bytes.restype = sz
        L.bp_csrmv_plan.argtypes = [P, P, P, i64, i64, i32, i32, P, sz,
                                    ctypes.POINTER(CsrmvPlanInfo), P, sz, P]
        L.bp_event_csrmv_planned.argtypes = [P, sz, ctypes.POINTER(CsrmvPlanInfo), P, P, P, f32,
                                             i64, i64, P, P, i32, u32, P, sz, P]
        jit_tail = [P, i64, i64, i64, i64, P, i32, u32, P, sz, P]
        L.bp_jitconn_event_mv_homo.argtypes = [ctypes.POINTER(JitConn), f32] + jit_tail
        L.bp_jitconn_event_mv_uniform.argtypes = [ctypes.POINTER(JitConn), f32, f32] + jit_tail
        L.bp_jitconn_event_mv_normal.argtypes = [ctypes.POINTER(JitConn), f32, f32] + jit_tail
        L.bp_jitconn_mv_homo.argtypes = [ctypes.POINTER(JitConn), f32, P] + jit_tail[1:]
        L.bp_jitconn_mv_uniform.argtypes = [ctypes.POINTER(JitConn), f32, f32, P] + jit_tail[1:]
        L.bp_jitconn_mv_normal.argtypes = [ctypes.POINTER(JitConn), f32, f32, P] + jit_tail[1:]
        L.bp_jitconn_row_counts.argtypes = [ctypes.POINTER(JitConn), i64, i64, P, P]
        L.bp_jitconn_indptr.argtypes = [ctypes.POINTER(JitConn), i64, i64, P, P]
        L.bp_jitconn_materialize.argtypes = [ctypes.POINTER(JitConn), i32, f32, f32,
                                             i64, i64, P, P, P, P]
        L.bp_neuron_step.argtypes = [ctypes.POINTER(NeuronParams),
                                     ctypes.POINTER(NeuronState), i64, P, P, P, i64, P]
        L.bp_network_workspace_bytes.argtypes = [ctypes.POINTER(NetworkDesc)]
        L.bp_network_workspace_bytes.restype = sz
        L.bp_network_create.argtypes = [ctypes.POINTER(NetworkDesc), P,
                                        ctypes.POINTER(ctypes.c_void_p)]
        L.bp_network_step.argtypes = [P, i64, P, P, P]
        L.bp_network_profile_begin.argtypes = [P, i64]
        L.bp_network_profile_end.argtypes = [P, P, P, P]
        L.bp_network_scatter.argtypes = [P, P]
        L.bp_network_update.argtypes = [P, P, P]
        L.bp_network_update_overlap.argtypes = [P, P, P, P]
        L.bp_network_counters.argtypes = [P, P, P]
        L.bp_network_destroy.argtypes = [P]
        L.bp_network_destroy.restype = None
        L.bp_network_describe.argtypes = [P, P, i32]
        L.bp_network_device_bytes.argtypes = [P]
        L.bp_network_device_bytes.restype = sz
        L.bp_nccl_unique_id.argtypes = [P]
        L.bp_nccl_version.argtypes = [P]
        for name in EXPORTED:
            if name not in ("bp_network_destroy", "bp_status_string",
                            "bp_last_error", "bp_conn_len", "bp_workspace_bytes",
                            "bp_csrmv_workspace_bytes", "bp_csrmv_plan_bytes",
                            "bp_jitconn_workspace_bytes",
                            "bp_network_workspace_bytes", "bp_abi_version",
                            "bp_network_device_bytes"):
                getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def _check(status: int):
    if status != 0:
        L = lib()
        raise BpError(f"{L.bp_status_string(status).decode()}: "
                      f"{L.bp_last_error().decode()}")


def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _out_kind(out: torch.Tensor) -> int:
    if out.dtype == torch.float32:
        return OUT_F32
    if out.dtype == torch.int64:
        return OUT_FIX64
    if out.dtype == torch.int32:
        return OUT_FIX32            # conductance state only (rule F2)
    raise BpError(f"output dtype {out.dtype}: float32, int64 or int32 (fixed point)")


def _cuda(*ts):
    for t in ts:
        if t is not None and (not t.is_cuda or not t.is_contiguous()):
            raise BpError("inputs must be contiguous CUDA tensors")


# ------------------------------------------------------------------ helpers

def conn_len(prob: float) -> int:
    return int(lib().bp_conn_len(float(prob)))


def workspace_bytes(n_rows: int) -> int:
    return int(lib().bp_workspace_bytes(int(n_rows)))


def workspace(n_rows: int, device=None) -> torch.Tensor:
    return torch.empty(workspace_bytes(n_rows), dtype=torch.uint8,
                       device=device or torch.cuda.current_device())


def jitconn_spec(seed: int, prob: float, conn_len: int = 0, seg_len: int = 0,
                 gap_law: int = GAP_UNIFORM) -> JitConn:
    """bp_jitconn; gap_law GAP_GEOMETRIC selects rule J10 (Geo(p) gaps)."""
    return JitConn(int(seed) & (2 ** 64 - 1), float(prob), int(conn_len), int(seg_len),
                   int(gap_law), 0)


# ------------------------------------------------------------- operators

def compact_spikes(spikes: torch.Tensor, n: int, active: torch.Tensor,
                   count: torch.Tensor, stream=None):
    _cuda(spikes, active, count)
    _check(lib().bp_compact_spikes(_ptr(spikes), int(n), _ptr(active),
                                   _ptr(count), _stream(stream)))


def event_csrmv(indptr, indices, data, w_homo, n_rows, n_cols, spikes, out,
                accumulate=False, ws=None, stream=None, plan=None):
    """brainpy.math.event.csrmv (Listing S1) -> out[n_cols] (f32 or fix64).
    plan: optional csrmv_plan(...) of this matrix (skips the per-call split)."""
    _cuda(indptr, indices, data, spikes, out)
    if ws is None:
        nbytes = int(lib().bp_csrmv_workspace_bytes(int(n_rows), int(n_cols), _out_kind(out)))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=out.device)
    tail = (_ptr(indptr), _ptr(indices), _ptr(data), float(w_homo), int(n_rows),
            int(n_cols), _ptr(spikes), _ptr(out), _out_kind(out),
            ACCUMULATE if accumulate else 0, _ptr(ws), ws.numel(), _stream(stream))
    if plan is not None:
        _check(lib().bp_event_csrmv_planned(_ptr(plan.buf), plan.buf.numel(),
                                            ctypes.byref(plan.info), *tail))
    else:
        _check(lib().bp_event_csrmv(*tail))
    return out


def csrmv_gather(indptr, indices, data, w_homo, n_rows, n_cols, spikes, out,
                 accumulate=False, stream=None):
    """Gather orientation (csrmv transpose=False, reading G1): out[r] (+)=
    sum over row r of w_k [spike indices[k]] -> out[n_rows] (f32 or fix64)."""
    _cuda(indptr, indices, data, spikes, out)
    _check(lib().bp_csrmv_gather(_ptr(indptr), _ptr(indices), _ptr(data), float(w_homo),
                                 int(n_rows), int(n_cols), _ptr(spikes), _ptr(out),
                                 _out_kind(out), ACCUMULATE if accumulate else 0,
                                 _stream(stream)))
    return out


def event_csrmv_grad(indptr, indices, data, w_homo, n_rows, n_cols, spikes, gy,
                     grad_data=None, grad_events=None, grad_w=None, stream=None):
    """Reverse mode of the event scatter y = M^T s (reading G1): fills the
    given outputs (grad_data[nnz] f32, grad_events[n_rows] f32, grad_w f64[1])."""
    _cuda(indptr, indices, data, spikes, gy, grad_data, grad_events, grad_w)
    _check(lib().bp_event_csrmv_grad(_ptr(indptr), _ptr(indices), _ptr(data), float(w_homo),
                                     int(n_rows), int(n_cols), _ptr(spikes), _ptr(gy),
                                     _ptr(grad_data), _ptr(grad_events), _ptr(grad_w),
                                     _stream(stream)))
    return grad_data, grad_events, grad_w


class CsrmvPlan:
    """A bp_csrmv_plan analysis: the device buffer and its host summary."""

    def __init__(self, buf, info):
        self.buf, self.info = buf, info

    @property
    def f32_fixed_bits(self) -> int:
        return int(self.info.f32_fixed_bits)


def csrmv_plan(indptr, indices, n_rows, n_cols, out_dtype=torch.float32, homo=True,
               data=None, stream=None):
    """Analysis of a matrix reused across calls (split points of every row at
    the column tiles; for heterogeneous weights with an fp32 output also the
    rule-T4 scale, which synchronises the stream once); pass the result as
    event_csrmv(..., plan=...).  None when there is nothing to precompute."""
    _cuda(indptr, indices, data)
    kind = 1 if out_dtype == torch.int64 else 0
    homo = bool(homo) and data is None
    nbytes = int(lib().bp_csrmv_plan_bytes(int(n_rows), int(n_cols), kind, int(homo)))
    if nbytes == 0:
        return None
    buf = torch.empty(nbytes, dtype=torch.uint8, device=indptr.device)
    ws = None
    if not homo:
        ws = torch.empty(int(lib().bp_csrmv_workspace_bytes(int(n_rows), int(n_cols), kind)),
                         dtype=torch.uint8, device=indptr.device)
    info = CsrmvPlanInfo()
    _check(lib().bp_csrmv_plan(_ptr(indptr), _ptr(indices), _ptr(data), int(n_rows), int(n_cols),
                               kind, int(homo), _ptr(buf), buf.numel(), ctypes.byref(info),
                               _ptr(ws), 0 if ws is None else ws.numel(), _stream(stream)))
    return CsrmvPlan(buf, info)


def jitconn_event_mv(law: int, spec: JitConn, w0: float, w1: float, spikes,
                     n_rows, n_cols, out, col_begin=0, col_end=None,
                     accumulate=False, ws=None, stream=None):
    """brainpy.math.jitconn.event_mv_prob_{homo,uniform,normal} (Listing S2)."""
    _cuda(spikes, out)
    col_end = n_cols if col_end is None else col_end
    if ws is None:
        nbytes = int(lib().bp_jitconn_workspace_bytes(int(n_rows), int(col_begin), int(col_end),
                                                      _out_kind(out)))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=out.device)
    flags = ACCUMULATE if accumulate else 0
    tail = (_ptr(spikes), int(n_rows), int(n_cols), int(col_begin), int(col_end),
            _ptr(out), _out_kind(out), flags, _ptr(ws), ws.numel(), _stream(stream))
    L = lib()
    if law == LAW_HOMO:
        st = L.bp_jitconn_event_mv_homo(ctypes.byref(spec), float(w0), *tail)
    elif law == LAW_UNIFORM:
        st = L.bp_jitconn_event_mv_uniform(ctypes.byref(spec), float(w0), float(w1), *tail)
    elif law == LAW_NORMAL:
        st = L.bp_jitconn_event_mv_normal(ctypes.byref(spec), float(w0), float(w1), *tail)
    else:
        raise BpError(f"unknown law {law}")
    _check(st)
    return out


def jitconn_mv(law: int, spec: JitConn, w0: float, w1: float, v, n_rows, n_cols, out,
               col_begin=0, col_end=None, accumulate=False, ws=None, stream=None):
    """brainpy.math.jitconn.mv_prob_{homo,uniform,normal}(vector, ...): the
    non-event product out[c] (+)= sum_r v[r] w_e (reading MV1)."""
    _cuda(v, out)
    col_end = n_cols if col_end is None else col_end
    if ws is None:
        nbytes = int(lib().bp_jitconn_workspace_bytes(int(n_rows), int(col_begin), int(col_end),
                                                      _out_kind(out)))
        ws = torch.empty(nbytes, dtype=torch.uint8, device=out.device)
    tail = (_ptr(v), int(n_rows), int(n_cols), int(col_begin), int(col_end), _ptr(out),
            _out_kind(out), ACCUMULATE if accumulate else 0, _ptr(ws), ws.numel(),
            _stream(stream))
    L = lib()
    if law == LAW_HOMO:
        _check(L.bp_jitconn_mv_homo(ctypes.byref(spec), float(w0), *tail))
    elif law == LAW_UNIFORM:
        _check(L.bp_jitconn_mv_uniform(ctypes.byref(spec), float(w0), float(w1), *tail))
    else:
        _check(L.bp_jitconn_mv_normal(ctypes.byref(spec), float(w0), float(w1), *tail))
    return out


def jitconn_event_mv_homo(spec, weight, spikes, n_rows, n_cols, out, **kw):
    return jitconn_event_mv(LAW_HOMO, spec, weight, 0.0, spikes, n_rows, n_cols, out, **kw)


def jitconn_event_mv_uniform(spec, w_low, w_high, spikes, n_rows, n_cols, out, **kw):
    return jitconn_event_mv(LAW_UNIFORM, spec, w_low, w_high, spikes, n_rows, n_cols, out, **kw)


def jitconn_event_mv_normal(spec, w_mu, w_sigma, spikes, n_rows, n_cols, out, **kw):
    return jitconn_event_mv(LAW_NORMAL, spec, w_mu, w_sigma, spikes, n_rows, n_cols, out, **kw)


def jitconn_materialize(spec: JitConn, n_rows: int, n_cols: int, law=LAW_HOMO,
                        w0=1.0, w1=0.0, with_data=True, device=None, stream=None):
    """CSR of the implied matrix, generated by the kernels' own generator."""
    device = device or torch.cuda.current_device()
    indptr = torch.empty(n_rows + 1, dtype=torch.int64, device=device)
    _check(lib().bp_jitconn_indptr(ctypes.byref(spec), int(n_rows), int(n_cols),
                                   _ptr(indptr), _stream(stream)))
    nnz = int(indptr[-1].item())
    indices = torch.empty(max(nnz, 1), dtype=torch.int32, device=device)
    data = torch.empty(max(nnz, 1), dtype=torch.float32, device=device) if with_data else None
    _check(lib().bp_jitconn_materialize(ctypes.byref(spec), int(law), float(w0),
                                        float(w1), int(n_rows), int(n_cols),
                                        _ptr(indptr), _ptr(indices), _ptr(data),
                                        _stream(stream)))
    return indptr, indices[:nnz], (data[:nnz] if data is not None else None)


# ------------------------------------------------------------- neurons

def lif_params(dt=0.1, tau=20.0, tau_e=5.0, tau_i=10.0, v_rest=-60.0,
               v_reset=-60.0, v_th=-50.0, r=1.0, i_ext=20.0, e_exc=0.0,
               e_inh=-80.0, tau_ref=5.0) -> NeuronParams:
    """LifRef + Expon + COBA of Listing S3, I_ext = 20."""
    p = NeuronParams()
    p.model = MODEL_LIF
    p.ref_steps = int(round(tau_ref / dt))
    p.v_rest, p.v_reset, p.v_th, p.r = v_rest, v_reset, v_th, r
    p.i_ext, p.e_exc, p.e_inh = i_ext, e_exc, e_inh
    p.alpha_v = float(ctypes.c_float(math.exp(-dt / tau)).value)
    p.alpha_e, p.alpha_i = math.exp(-dt / tau_e), math.exp(-dt / tau_i)
    return p


def hh_params(dt=0.1, tau_e=5.0, tau_i=10.0, i_ext=0.0) -> NeuronParams:
    """COBA-HH (Brette et al. 2007 benchmark 3; rule H1, EXTERNAL)."""
    p = NeuronParams()
    p.model = MODEL_HH
    p.c_m, p.g_l, p.e_l = 200.0, 10.0, -60.0
    p.g_na, p.e_na, p.g_k, p.e_k, p.v_t = 20000.0, 50.0, 6000.0, -90.0, -63.0
    p.e_exc, p.e_inh, p.i_ext, p.dt, p.v_spike = 0.0, -80.0, i_ext, dt, -20.0
    p.alpha_e, p.alpha_i = math.exp(-dt / tau_e), math.exp(-dt / tau_i)
    return p


def _state_struct(state: dict) -> NeuronState:
    g = state["g_e"]
    s = NeuronState()
    s.v = state["v"].data_ptr()
    s.g_exc = g.data_ptr()
    s.g_inh = state["g_i"].data_ptr()
    s.g_kind = _out_kind(g)
    s.g_frac_bits = int(state.get("frac_bits", 0))
    for k, f in (("ref", "ref"), ("m", "m"), ("h", "h"), ("n", "n_gate")):
        if state.get(k) is not None:
            setattr(s, f, state[k].data_ptr())
    return s


def neuron_step(params: NeuronParams, state: dict, spikes_out: torch.Tensor,
                active=None, count=None, active_base=0, stream=None):
    """One fused Expon + COBA + LIF/HH step of all neurons in `state`."""
    n = state["v"].numel()
    _check(lib().bp_neuron_step(ctypes.byref(params), ctypes.byref(_state_struct(state)),
                                n, _ptr(spikes_out), _ptr(active), _ptr(count),
                                int(active_base), _stream(stream)))


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for BP_EXCHANGE_NCCL networks (bp_nccl_unique_id)."""
    buf = (ctypes.c_uint8 * 128)()
    _check(lib().bp_nccl_unique_id(ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def nccl_version() -> int | None:
    """NCCL version code the library resolves, or None when NCCL cannot be
    loaded (bp_nccl_version)."""
    v = ctypes.c_int32()
    if lib().bp_nccl_version(ctypes.byref(v)) != 0:
        return None
    return int(v.value)


def projection(*, pre_begin, pre_end, weight, receptor=RECEPTOR_EXC, jit=None, csr=None):
    """One bp_projection: rows = neurons [pre_begin, pre_end), `weight` per
    event into the receptor's conductance; jit=JitConn or csr=(indptr,
    indices) (column-sliced to this process's columns)."""
    p = Projection()
    p.receptor = int(receptor)
    p.pre_begin, p.pre_end = int(pre_begin), int(pre_end)
    p.weight = float(weight)
    if jit is not None:
        p.conn = CONN_JIT
        p.jit = jit
    else:
        ip, ix = csr[0], csr[1]
        _cuda(ip, ix)
        if ip.dtype != torch.int64 or ix.dtype != torch.int32:
            raise BpError("CSR projection: indptr int64, indices int32")
        if ip.numel() != int(pre_end) - int(pre_begin) + 1:
            raise BpError("CSR projection: indptr must have pre_end - pre_begin + 1 entries")
        p.conn = CONN_CSR
        p.indptr, p.indices = ip.data_ptr(), ix.data_ptr()
    return p


def _check_buf(t, numel, dtype, device, what, host_ok=False):
    """A caller buffer the library writes: right dtype, contiguous, large
    enough, and on the network's device (or pinned host memory when
    host_ok)."""
    if t is None:
        return
    if t.dtype != dtype or not t.is_contiguous() or t.numel() < numel:
        raise BpError(f"{what}: need >= {numel} contiguous {dtype} elements")
    if t.is_cuda:
        if t.device != device:
            raise BpError(f"{what}: on {t.device}, the network is on {device}")
    elif not (host_ok and t.is_pinned()):
        raise BpError(f"{what}: must be a CUDA tensor" + (" or pinned host memory"
                                                          if host_ok else ""))


class Network:
    """Handle over bp_network_* (Listing S3's update loop, rule S1, with up to
    MAX_PROJ projections merged per receptor).

    Keeps references to every tensor whose pointer it passed to the library.
    """

    def __init__(self, *, model, n, state: dict, spikes, params, projections,
                 col_begin=0, col_end=None, stream=None, delay=1, keep=(),
                 exchange=EXCHANGE_CALLER, rank=0, world=1, part_len=0, nccl_id=None,
                 ws=None):
        col_end = n if col_end is None else col_end
        if not 1 <= len(projections) <= MAX_PROJ:
            raise BpError(f"1..{MAX_PROJ} projections, got {len(projections)}")
        d = NetworkDesc()
        d.model = model
        d.delay_steps = int(delay)
        d.g_kind = _out_kind(state["g_e"])
        d.n, d.col_begin, d.col_end = n, col_begin, col_end
        d.n_proj = len(projections)
        for k, p in enumerate(projections):
            d.proj[k] = p
        self._keep = [state, spikes, *keep]
        d.params = params
        d.state = _state_struct(state)
        d.spikes = spikes.data_ptr()
        d.exchange, d.rank, d.world, d.part_len = int(exchange), int(rank), int(world), int(part_len)
        if nccl_id is not None:
            ctypes.memmove(d.nccl_id, nccl_id, 128)
        nbytes = int(lib().bp_network_workspace_bytes(ctypes.byref(d)))
        if ws is None:
            ws = torch.zeros(nbytes, dtype=torch.uint8, device=spikes.device)
        _check_buf(ws, nbytes, torch.uint8, spikes.device, "ws")
        self.ws = ws
        d.ws, d.ws_bytes = ws.data_ptr(), ws.numel()
        self.desc = d
        self.device = spikes.device
        self.state, self.spikes = state, spikes
        self.n_local = col_end - col_begin
        self.local_words = (self.n_local + 31) // 32
        handle = ctypes.c_void_p()
        _check(lib().bp_network_create(ctypes.byref(d), _stream(stream),
                                       ctypes.byref(handle)))
        self._h = handle

    def step(self, n_steps: int, raster=None, counts=None, stream=None):
        """raster: device int32 [n_steps, local_words] (nullable); counts:
        device or pinned host int32 [n_steps] (nullable)."""
        _check_buf(raster, int(n_steps) * self.local_words, torch.int32, self.device, "raster")
        _check_buf(counts, int(n_steps), torch.int32, self.device, "counts", host_ok=True)
        _check(lib().bp_network_step(self._h, int(n_steps), _ptr(raster), _ptr(counts),
                                     _stream(stream)))

    def profile_begin(self, max_steps: int):
        _check(lib().bp_network_profile_begin(self._h, int(max_steps)))

    def profile_end(self):
        """-> (scatter_ms_total, update_ms_total, steps) over the recorded steps."""
        sc, up, n = ctypes.c_double(), ctypes.c_double(), ctypes.c_int64()
        _check(lib().bp_network_profile_end(self._h, ctypes.byref(sc), ctypes.byref(up),
                                            ctypes.byref(n)))
        return sc.value, up.value, n.value

    def scatter(self, stream=None):
        _check(lib().bp_network_scatter(self._h, _stream(stream)))

    def update(self, raster_row=None, stream=None):
        _check_buf(raster_row, self.local_words, torch.int32, self.device, "raster_row")
        _check(lib().bp_network_update(self._h, _ptr(raster_row), _stream(stream)))

    def update_overlap(self, exchange_stream, raster_row=None, stream=None):
        """update(); `exchange_stream` (torch.cuda.Stream) waits for this
        step's spike words only, so an all-gather there overlaps the local
        binning kernel."""
        _check_buf(raster_row, self.local_words, torch.int32, self.device, "raster_row")
        _check(lib().bp_network_update_overlap(self._h, _ptr(raster_row), _stream(stream),
                                               _stream(exchange_stream)))

    def counters(self, stream=None):
        """-> (local spikes, synaptic events delivered, saturated FIX32 updates)."""
        return self.counters_all(stream)[:3]

    def counters_all(self, stream=None):
        """-> (spikes, events, saturated FIX32 updates, non-finite V seen with
        BP_DEBUG_NAN=1)."""
        out = (ctypes.c_uint64 * 4)()
        _check(lib().bp_network_counters(self._h, ctypes.cast(out, ctypes.c_void_p),
                                         _stream(stream)))
        return tuple(int(x) for x in out)

    def device_bytes(self) -> int:
        """Device memory the library allocated for this network (buckets,
        projection table)."""
        return int(lib().bp_network_device_bytes(self._h))

    def describe(self) -> dict:
        """The execution plan chosen at create (bp_network_describe)."""
        out = (ctypes.c_int32 * 8)()
        _check(lib().bp_network_describe(self._h, ctypes.cast(out, ctypes.c_void_p), 8))
        keys = ("small", "dense", "n_tiles", "cap", "fold_classes", "bin_lanes", "nccl",
                "classes")
        return dict(zip(keys, (int(x) for x in out)))

    def close(self):
        if getattr(self, "_h", None) is not None and self._h.value:
            lib().bp_network_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
