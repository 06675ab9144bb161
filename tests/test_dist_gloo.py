"""Multi-process host logic of the postsynaptic partition on CPU.

Two ranks over torch.distributed/gloo run the partition arithmetic and the
bit-packed spike all-gather of paper_2311_05106_b200.network (the same
functions the NCCL path uses); the per-rank local compute is the CPU oracle
restricted to the rank's columns.  The gathered rasters must equal the
single-process network bit for bit (fixed point) -- no cross-rank
reduction exists, so partitioning cannot change any value.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_05106_b200 import inputs
from paper_2311_05106_b200.network import SEED_E, SEED_I, exchange_spikes, partition

N, STEPS = 3000, 120


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _specs(orc, n, seg_len):
    K = orc.conn_len(80.0 / n)
    je = orc.JitSpec(SEED_E, K, seg_len, orc.LAW_HOMO, 0.6)
    ji = orc.JitSpec(SEED_I, K, seg_len, orc.LAW_HOMO, 6.7)
    return je, ji


def _rank_main(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import oracle
    part = partition(N, world, rank)
    lo, hi = part.col_begin, part.col_end
    je, ji = _specs(oracle, N, part.local)
    n_exc = N * 4 // 5
    v0 = inputs.lif_v0(N)
    st = dict(v=v0[lo:hi].copy(), g_e=np.zeros(hi - lo, np.int64),
              g_i=np.zeros(hi - lo, np.int64), ref=np.zeros(hi - lo, np.uint8))
    words = torch.zeros(part.padded_words, dtype=torch.int32)
    params = oracle.lif_params()
    raster = []
    for _ in range(STEPS):
        spikes = inputs.unpack_bits(words.numpy().view(np.uint32), N)
        oracle.jit_event_mv(je, n_exc, N, spikes[:n_exc], lo, hi, oracle.OUT_FIX, out=st["g_e"])
        oracle.jit_event_mv(ji, N - n_exc, N, spikes[n_exc:], lo, hi, oracle.OUT_FIX, out=st["g_i"])
        local = oracle.lif_step(params, st["v"], st["g_e"], st["g_i"], st["ref"])
        mine = np.zeros(part.local, np.uint8)
        mine[:hi - lo] = local
        lw = part.local_words
        words[rank * lw:(rank + 1) * lw] = torch.from_numpy(inputs.pack_bits(mine).view(np.int32))
        exchange_spikes(words, part)
        raster.append(inputs.unpack_bits(words.numpy().view(np.uint32), N))
    np.save(os.path.join(out_dir, f"raster_{rank}.npy"), np.stack(raster))
    np.save(os.path.join(out_dir, f"v_{rank}.npy"), st["v"])
    dist.barrier()
    dist.destroy_process_group()


def test_partition_arithmetic():
    for n, world in [(3000, 2), (12_500_000 * 8, 8), (4097, 4), (100, 3)]:
        parts = [partition(n, world, r) for r in range(world)]
        assert parts[0].col_begin == 0 and parts[-1].col_end == n
        for a, b in zip(parts, parts[1:]):
            assert a.col_end == b.col_begin
        for p in parts:
            # a rank past the end owns an empty slice [n, n)
            assert (p.col_begin % 32 == 0 or p.col_begin == n) and p.local % 32 == 0
            assert p.padded_words * 32 >= n
    p = partition(1000, 4, 1, align=100)
    assert p.local % 800 == 0          # lcm(32, 100) = 800


@pytest.mark.timeout(600)
def test_two_rank_gloo_equals_single_process(orc, tmp_path):
    world = 2
    port = _free_port()
    mp.start_processes(_rank_main, args=(world, port, str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    raster = [np.load(tmp_path / f"raster_{r}.npy") for r in range(world)]
    assert np.array_equal(raster[0], raster[1])          # every rank sees all spikes
    # single-process reference with the same segment grid (rule J4)
    local = partition(N, world, 0).local
    je, ji = _specs(orc, N, local)
    n_exc = N * 4 // 5
    st = dict(v=inputs.lif_v0(N), g_e=np.zeros(N, np.int64), g_i=np.zeros(N, np.int64),
              ref=np.zeros(N, np.uint8), spikes=np.zeros(N, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, orc.Projection(0, n_exc, jit=je),
                           orc.Projection(n_exc, N - n_exc, jit=ji), STEPS)
    assert want.sum() > 0
    assert np.array_equal(raster[0], want)
    v = np.concatenate([np.load(tmp_path / f"v_{r}.npy") for r in range(world)])
    assert np.array_equal(v.view(np.uint32), st["v"].view(np.uint32))


def _id_rank(rank, world, port, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2311_05106_b200.network import share_nccl_id
    # rank 0's id (a stand-in for bp_nccl_unique_id: no GPU here) reaches every rank
    got = share_nccl_id(rank, world, make_id=lambda: bytes(range(128)))
    with open(os.path.join(out_dir, f"id_{rank}.bin"), "wb") as f:
        f.write(got)
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_nccl_id_reaches_every_rank(tmp_path):
    """BP_EXCHANGE_NCCL setup (network.share_nccl_id): rank 0 creates the
    128-byte ncclUniqueId and the process group broadcasts it, so every
    rank's bp_network_create gets the same bytes."""
    world = 3
    mp.start_processes(_id_rank, args=(world, _free_port(), str(tmp_path)), nprocs=world,
                       join=True, start_method="spawn")
    ids = [(tmp_path / f"id_{r}.bin").read_bytes() for r in range(world)]
    assert all(i == bytes(range(128)) for i in ids)
