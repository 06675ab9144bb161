"""The multi-process network path ON THE GPU: two ranks (processes) share
cuda:0 and exchange the bit-packed spikes through torch.distributed/gloo (the
all-gather is host-mediated, so no kernel of one rank waits on the other).
bp_network_update / bp_network_scatter (remote-word compaction + binning)
must reproduce the single-process oracle bit for bit.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2311_05106_b200 import inputs
from paper_2311_05106_b200.network import SEED_E, SEED_I, CobaNetwork, partition

pytestmark = pytest.mark.gpu

N, STEPS = 8192, 300


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _rank(rank, world, port, out_dir, mode, overlap):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import __graft_entry__ as ge
    ge.build_lib()
    torch.cuda.set_device(0)
    net = CobaNetwork(N, conn="jit", fixed=mode, rank=rank, world=world, device="cuda:0")
    rows = []
    for _ in range(STEPS):
        net.step_distributed(overlap=overlap)
        rows.append(net.spikes.cpu().numpy().view(np.uint32).copy())
    np.save(os.path.join(out_dir, f"r{rank}.npy"), np.stack(rows))
    np.save(os.path.join(out_dir, f"v{rank}.npy"), net.state["v"].cpu().numpy())
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(900)
@pytest.mark.parametrize("mode,overlap", [("fix32", True), ("f32", True), ("f32", False)])
def test_two_ranks_on_one_gpu_gloo(orc, tmp_path, mode, overlap):
    """overlap: the all-gather runs on a side stream that waits only for the
    update kernel (bp_network_update_overlap), concurrent with the binning."""
    world = 2
    mp.start_processes(_rank, args=(world, _free_port(), str(tmp_path), mode, overlap),
                       nprocs=world,
                       join=True, start_method="spawn")
    r0, r1 = np.load(tmp_path / "r0.npy"), np.load(tmp_path / "r1.npy")
    assert np.array_equal(r0, r1)
    local = partition(N, world, 0).local
    n_exc = N * 4 // 5
    K = orc.conn_len(80.0 / N)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, local, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, N - n_exc, jit=orc.JitSpec(SEED_I, K, local, orc.LAW_HOMO, 6.7))
    g = np.int32 if mode == "fix32" else np.float32
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(N), g_e=np.zeros(N, g), g_i=np.zeros(N, g),
              ref=np.zeros(N, np.uint8), spikes=np.zeros(N, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, STEPS)
    assert want.sum() > 0
    got = np.stack([inputs.unpack_bits(w, N) for w in r0])
    assert np.array_equal(got, want)
    v = np.concatenate([np.load(tmp_path / "v0.npy"), np.load(tmp_path / "v1.npy")])
    assert np.array_equal(v.view(np.uint32), st["v"].view(np.uint32))


def _graph_rank(rank, world, port, out_dir):
    """NCCL with one rank: the captured CUDA graph of step_distributed
    (network.capture, the N > 1 bench loop) against the eager loop."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", 0))
    import __graft_entry__ as ge
    ge.build_lib()
    out = {}
    for arm in ("graph", "eager"):
        net = CobaNetwork(N, conn="jit", fixed="fix32", rank=0, world=1, device="cuda:0")
        for _ in range(20):
            net.step_distributed()
        if arm == "graph":
            g, period = net.capture()
            for _ in range(200 // period):
                g.replay()
        else:
            for _ in range(200):
                net.step_distributed()
        torch.cuda.synchronize()
        out[arm + "_v"] = net.state["v"].cpu().numpy()
        out[arm + "_ge"] = net.state["g_e"].cpu().numpy()
        out[arm + "_spikes"] = np.array(net.counters()[:2], np.int64)
    np.savez(os.path.join(out_dir, "graph.npz"), **out)
    dist.destroy_process_group()


@pytest.mark.timeout(600)
def test_captured_distributed_step_equals_eager(orc, tmp_path):
    mp.start_processes(_graph_rank, args=(1, _free_port(), str(tmp_path)), nprocs=1,
                       join=True, start_method="spawn")
    d = np.load(tmp_path / "graph.npz")
    assert np.array_equal(d["graph_v"].view(np.uint32), d["eager_v"].view(np.uint32))
    assert np.array_equal(d["graph_ge"], d["eager_ge"])
    assert np.array_equal(d["graph_spikes"], d["eager_spikes"])
    assert d["eager_spikes"][0] > 0
    # and the oracle (rule S1, fix32) after the same 220 steps
    n_exc = N * 4 // 5
    K = orc.conn_len(80.0 / N)
    pe = orc.Projection(0, n_exc, jit=orc.JitSpec(SEED_E, K, N, orc.LAW_HOMO, 0.6))
    pi = orc.Projection(n_exc, N - n_exc, jit=orc.JitSpec(SEED_I, K, N, orc.LAW_HOMO, 6.7))
    orc.set_fix32_bits(20)
    st = dict(v=inputs.lif_v0(N), g_e=np.zeros(N, np.int32), g_i=np.zeros(N, np.int32),
              ref=np.zeros(N, np.uint8), spikes=np.zeros(N, np.uint8))
    want = orc.run_network("lif", orc.lif_params(), st, pe, pi, 220)
    assert int(want.sum()) == int(d["eager_spikes"][0])
    assert np.array_equal(d["eager_v"].view(np.uint32), st["v"].view(np.uint32))
