"""CPU-side checks of the C ABI: the library builds for sm_100a, loads, and
exports every symbol include/bp.h declares; host-only functions agree with
the oracle's rules; device calls fail loudly (no CPU fallback) without a GPU.
"""
import ctypes
import os
import re
import subprocess

import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def libbp():
    import __graft_entry__ as ge
    ge.build_lib()
    from paper_2311_05106_b200 import _binding
    return _binding.lib()


def _declared():
    src = open(os.path.join(ROOT, "include", "bp.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(bp_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_north_star_calls():
    names = _declared()
    for n in ("bp_event_csrmv", "bp_jitconn_event_mv_homo", "bp_jitconn_event_mv_uniform",
              "bp_jitconn_event_mv_normal", "bp_neuron_step", "bp_network_step"):
        assert n in names


def test_every_declared_symbol_is_exported(libbp):
    from paper_2311_05106_b200 import _binding
    out = subprocess.check_output(["nm", "-D", "--defined-only", _binding.LIB_PATH]).decode()
    exported = set(re.findall(r"\bT (bp_[a-z0-9_]+)", out))
    missing = [n for n in _declared() if n not in exported]
    assert not missing, missing
    assert set(_binding.EXPORTED) <= exported


def test_sass_is_sm100a():
    from paper_2311_05106_b200 import _binding
    out = subprocess.check_output(["cuobjdump", "--list-elf", _binding.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_conn_len_matches_oracle(libbp, orc):
    for p in [1e-3, 1e-2, 2e-2, 5e-2, 80 / 4e6, 80 / 1e8, 80 / 12.5e6, 0.6, 1.0,
              0.3333, 0.0, 1.5, float("nan")]:
        assert libbp.bp_conn_len(p) == orc.conn_len(p), p


def test_workspace_bytes(libbp):
    assert libbp.bp_workspace_bytes(0) == 256
    assert libbp.bp_workspace_bytes(100) >= 256 + 400
    assert libbp.bp_workspace_bytes(100) % 256 == 0


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU failure path")
def test_device_calls_fail_loudly_without_gpu(libbp):
    rc = libbp.bp_compact_spikes(None, 0, None, ctypes.c_void_p(16), None)
    assert rc != 0
    assert libbp.bp_last_error()


def test_struct_layouts_match_the_header(tmp_path):
    """The ctypes mirrors of bp.h's structs have the C layout (size and the
    offsets of the fields the binding sets), checked against gcc."""
    from paper_2311_05106_b200 import _binding as B
    fields = {"bp_network_desc": (B.NetworkDesc, ["n", "col_begin", "proj", "params", "state",
                                                  "spikes", "ws_bytes", "exchange",
                                                  "part_len", "nccl_id"]),
              "bp_projection": (B.Projection, ["pre_begin", "weight", "jit", "indptr"]),
              "bp_jitconn": (B.JitConn, ["prob", "seg_len", "gap_law"]),
              "bp_neuron_params": (B.NeuronParams, ["alpha_e", "c_m", "v_spike"]),
              "bp_neuron_state": (B.NeuronState, ["g_kind", "ref", "n_gate"])}
    src = ['#include <stdio.h>', '#include <stddef.h>', '#include "bp.h"', "int main(void) {"]
    for cname, (_, fs) in fields.items():
        src.append(f'  printf("{cname} %zu\\n", sizeof({cname}));')
        for f in fs:
            src.append(f'  printf("{cname}.{f} %zu\\n", offsetof({cname}, {f}));')
    src.append("  return 0; }")
    c = tmp_path / "layout.c"
    c.write_text("\n".join(src))
    exe = tmp_path / "layout"
    subprocess.check_call(["gcc", "-I", os.path.join(ROOT, "include"), str(c), "-o", str(exe)])
    got = dict(line.split() for line in subprocess.check_output([str(exe)]).decode().splitlines())
    for cname, (cls, fs) in fields.items():
        assert int(got[cname]) == ctypes.sizeof(cls), cname
        for f in fs:
            assert int(got[f"{cname}.{f}"]) == getattr(cls, f).offset, (cname, f)


def test_library_has_no_link_time_nccl_dependency(libbp):
    """NCCL is resolved at run time (dlopen): loading libbp.so never pulls a
    second libnccl into a process that already has torch's."""
    from paper_2311_05106_b200 import _binding
    out = subprocess.check_output(["readelf", "-d", _binding.LIB_PATH]).decode()
    assert "nccl" not in out


def test_nccl_resolves_at_run_time(libbp):
    """bp_nccl_version: the library finds an NCCL (torch's, already in the
    process) without a link-time dependency; a version code >= 2.27."""
    import paper_2311_05106_b200 as bp
    v = bp.nccl_version()
    assert v is not None and v >= 22700
