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
