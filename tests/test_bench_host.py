"""Host logic of bench.py (CPU): workload parameters, incl. the Fig S3B/S3C
weight rescaling of reading R29 (w = w_80 * 80 / fan-in)."""
import math

import pytest

import bench


def test_default_workload_is_config5():
    p, we, wi = bench.net_params("coba_lif_jit", bench.network_size("coba_lif_jit", 1))
    assert bench.network_size("coba_lif_jit", 8) == 8 * bench.N_PER_GPU
    assert math.isclose(p * bench.N_PER_GPU, 80.0) and (we, wi) == (0.6, 6.7)


@pytest.mark.parametrize("wl,fan_in", [("coba4m_k1000", 1000.0), ("coba4m_p001", 4000.0)])
def test_fig_s3_weights_keep_the_mean_drive(wl, fan_in):
    n = bench.network_size(wl, 1)
    p, we, wi = bench.net_params(wl, n)
    assert math.isclose(p * n, fan_in)
    # K w is the 80-synapse network's: 80 * 0.6 and 80 * 6.7
    assert math.isclose(p * n * we, 80 * 0.6) and math.isclose(p * n * wi, 80 * 6.7)


def test_hh_weights_and_small_network():
    p, we, wi = bench.net_params("hh400k_csr", 400_000)
    assert (we, wi) == (6.0, 67.0) and math.isclose(p * 400_000, 80.0)
    assert bench.network_size("coba4000_csr", 8) == 4000       # strong scaling: fixed size
