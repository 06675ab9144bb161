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


@pytest.mark.parametrize("wl", ["coba4m_jit", "coba4m_k1000", "coba4m_p001", "coba100m_jit"])
def test_strong_scaling_connectivity_is_the_same_at_every_gpu_count(wl):
    """Strong-scaling JIT configs use seg_len = n / 8 at EVERY G, so the
    partition at G = 1, 2, 4, 8 falls on segment boundaries and the JIT
    matrix (a function of seed, K, seg_len, n only: rule J4) is the same."""
    from paper_2311_05106_b200.network import partition
    n = bench.network_size(wl, 1)
    L = bench.seg_len_of(wl, n)
    assert L % 32 == 0 and 8 * L >= n
    for g in (1, 2, 4, 8):
        assert bench.network_size(wl, g) == n
        for r in range(g):
            part = partition(n, g, r, align=L)
            assert part.col_begin % L == 0
            assert part.col_end == n or part.col_end % L == 0


def test_weak_scaling_segment_is_one_gpu():
    for g in (1, 2, 4, 8):
        n = bench.network_size("coba_lif_jit", g)
        assert bench.seg_len_of("coba_lif_jit", n) == bench.N_PER_GPU


def test_settle_default():
    assert bench.settle_default("coba_lif_jit") == 2000
    assert bench.settle_default("coba4000_csr") == 0


def test_launches_per_step():
    # config 5 at G = 1: k_step + k_bin; G = 8: + compaction + remote binning
    assert bench.launches_per_step("lif", 12_500_000, 12_500_000, 1) == 2
    assert bench.launches_per_step("lif", 12_500_000, 100_000_000, 8) == 4
    # config 3 strong scaling at G = 8: remote words listed by the binning
    assert bench.launches_per_step("lif", 500_000, 4_000_000, 8) == 3
    # config 4: the dense HH update delivers its own spikes
    assert bench.launches_per_step("hh", 400_000, 400_000, 1) == 1
    assert bench.launches_per_step("hh", 200_000, 400_000, 2) == 2
