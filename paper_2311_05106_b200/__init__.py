"""B200-native event-driven synaptic projection library (BrainPy hot path).

Public API = the C ABI of include/bp.h, reached through the thin ctypes
binding in _binding.py (argument marshalling only), plus the network/host
logic in network.py.  libbp.so is loaded lazily on first use and its absence
raises; there is no CPU fallback.
"""
from ._binding import (ACCUMULATE, CONN_CSR, CONN_JIT, EXCHANGE_CALLER,  # noqa: F401
                       EXCHANGE_NCCL, GAP_GEOMETRIC, GAP_UNIFORM, MAX_PROJ,
                       RECEPTOR_EXC, RECEPTOR_INH, LAW_HOMO, LAW_NORMAL,
                       LAW_UNIFORM, MODEL_HH, MODEL_LIF, OUT_F32, OUT_FIX64,
                       BpError, JitConn, Network, NeuronParams, compact_spikes,
                       conn_len, csrmv_gather, csrmv_plan, event_csrmv, event_csrmv_grad, hh_params, jitconn_event_mv, jitconn_mv,
                       jitconn_event_mv_homo, jitconn_event_mv_normal,
                       jitconn_event_mv_uniform, jitconn_materialize,
                       jitconn_spec, lib, lif_params, nccl_unique_id, nccl_version, neuron_step,
                       projection, workspace, workspace_bytes)
