"""COBA E/I networks of Listing S3 on the C ABI, one process per GPU.

Host logic only: building the state tensors, the postsynaptic partition of
SURVEY 8(e) (rank g owns neurons [lo_g, hi_g)), and the per-step bit-packed
spike all-gather over torch.distributed (NCCL on GPUs, gloo in the CPU
tests).  Every arithmetic step of the simulation runs in libbp.so.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import torch

from . import _binding as B
from . import inputs

# Listing S3: 80 % excitatory, p = 80 / N, w_E = 0.6, w_I = 6.7.
SEED_E, SEED_I = 0x5EED0001, 0x5EED0002
W_E_LIF, W_I_LIF = 0.6, 6.7
W_E_HH, W_I_HH = 6.0, 67.0          # COBA-HH nS (rule H1, EXTERNAL)
# rule F2 fractional bits: LIF g stays < 2^11 (range 2048), HH g (nS) < 2^15
FIX32_BITS = {"lif": 20, "hh": 16}


@dataclass(frozen=True)
class Partition:
    """Postsynaptic slice [col_begin, col_end) of rank `rank` out of `world`.
    Every rank owns `local` neurons (the last one possibly fewer); `local`
    is a multiple of `align` (32-bit spike words, JIT segments)."""
    rank: int
    world: int
    n: int
    local: int

    @property
    def col_begin(self) -> int:
        return min(self.n, self.rank * self.local)

    @property
    def col_end(self) -> int:
        return min(self.n, (self.rank + 1) * self.local)

    @property
    def local_words(self) -> int:
        return self.local // 32

    @property
    def padded_words(self) -> int:
        """Length of the all-gathered spike vector in words (world * local/32)."""
        return self.world * self.local_words


def partition(n: int, world: int, rank: int, align: int = 32) -> Partition:
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"rank {rank} of world {world}")
    align = math.lcm(32, int(align))
    local = -(-n // world)
    local = -(-local // align) * align
    return Partition(rank, world, n, local)


def exchange_spikes(words: torch.Tensor, part: Partition, group=None,
                    send: torch.Tensor | None = None) -> torch.Tensor:
    """All-gather the bit-packed spike vector: rank g contributes its words
    [g*local/32, (g+1)*local/32) of `words` (length part.padded_words) and
    receives everybody else's (a8; "gather only non-zero spikes",
    realised as bit packing).  Works with NCCL and gloo."""
    import torch.distributed as dist
    lw = part.local_words
    mine = words[part.rank * lw:(part.rank + 1) * lw]
    if send is None:
        send = mine.clone()
    else:
        send.copy_(mine)
    dist.all_gather_into_tensor(words, send, group=group)
    return words


def share_nccl_id(rank: int, world: int, group=None, make_id=None) -> bytes:
    """The 128-byte ncclUniqueId of a BP_EXCHANGE_NCCL network: rank 0 makes
    it (bp_nccl_unique_id), every rank receives the same bytes over the
    torch.distributed process group (any backend)."""
    make_id = make_id or B.nccl_unique_id
    nccl_id = make_id() if rank == 0 else None
    if world > 1:
        import torch.distributed as dist
        obj = [nccl_id]
        dist.broadcast_object_list(obj, src=0, group=group)
        nccl_id = obj[0]
    if not isinstance(nccl_id, (bytes, bytearray)) or len(nccl_id) != 128:
        raise ValueError("ncclUniqueId must be 128 bytes")
    return bytes(nccl_id)


@dataclass(frozen=True)
class ProjSpec:
    """One projection of a network (bp_projection): the spikes of neurons
    [pre_begin, pre_end) add `weight` per event into the conductance of
    `receptor` ('exc' or 'inh') at their targets among all n neurons.
    Connectivity: JIT (seed, p, seg_len; event_mv_prob_homo) or a
    full CSR (indptr, indices) over the projection's rows (this rank keeps
    the columns it owns)."""
    pre_begin: int
    pre_end: int
    receptor: str
    weight: float
    seed: int | None = None
    p: float | None = None
    csr: tuple | None = None


class CobaNetwork:
    """One rank's share of the Listing S3 E/I network (COBA-LIF or COBA-HH),
    or of any network of up to 8 projections merged per receptor
    (`projections`, AlignPost P:130).

    conn='jit': connectivity regenerated each step from (seed, p) -- the
    EventJitFPHomoLinear / event_mv_prob_homo projection of P:973-981.
    conn='csr': stored CSR (event_csrmv, Listing S1); `csr` gives the full
    (indptr, indices) of the E rows and the I rows (torch CPU or CUDA), and
    this rank keeps the columns it owns.
    exchange='caller' (default): with world > 1 the spike all-gather runs in
    step_distributed through torch.distributed (NCCL or gloo); 'nccl': the
    library owns an NCCL communicator and run() executes whole steps,
    the all-gather included (bp_network_step; needs torch.distributed
    initialised when world > 1, only to broadcast the NCCL id).
    """

    def __init__(self, n: int, *, model: str = "lif", conn: str = "jit",
                 fixed: bool = True, p: float | None = None, seg_len: int | None = None,
                 rank: int = 0, world: int = 1, device=None, csr=None,
                 w_exc: float | None = None, w_inh: float | None = None,
                 seed_e: int = SEED_E, seed_i: int = SEED_I, v0=None,
                 init_seed: int = inputs.V0_SEED, spikes: torch.Tensor | None = None,
                 frac_bits: int | None = None, delay: int = 1,
                 projections: list[ProjSpec] | None = None, exchange: str = "caller",
                 group=None):
        device = torch.device(device or "cuda")
        self.n = n
        self.n_exc = n * 4 // 5
        self.model, self.conn, self.fixed = model, conn, fixed
        self.p = 80.0 / n if p is None else p
        if seg_len is None:
            # one JIT segment per rank: the partition is the segment (8(e))
            seg_len = partition(n, world, rank).local if world > 1 else n
        self.seg_len = seg_len
        self.part = partition(n, world, rank, align=seg_len if world > 1 else 32)
        lo, hi = self.part.col_begin, self.part.col_end
        n_local = hi - lo
        if model == "lif":
            w_exc = W_E_LIF if w_exc is None else w_exc
            w_inh = W_I_LIF if w_inh is None else w_inh
            params = B.lif_params()
        else:
            w_exc = W_E_HH if w_exc is None else w_exc
            w_inh = W_I_HH if w_inh is None else w_inh
            params = B.hh_params()
        self.w_exc, self.w_inh, self.params = w_exc, w_inh, params
        # conductance kind: fixed=True/"fix64" -> int64 2^-32 (rule F1),
        # "fix32" -> int32 2^-F (rule F2; F = 20 LIF, 16 HH), False/"f32" -> fp32
        mode = {True: "fix64", False: "f32"}.get(fixed, fixed)
        if mode not in ("fix64", "fix32", "f32"):
            raise ValueError(f"fixed={fixed!r}")
        self.mode = mode
        g_dtype = {"fix64": torch.int64, "fix32": torch.int32, "f32": torch.float32}[mode]
        st = {"g_e": torch.zeros(n_local, dtype=g_dtype, device=device),
              "g_i": torch.zeros(n_local, dtype=g_dtype, device=device)}
        if mode == "fix32":
            st["frac_bits"] = FIX32_BITS[model] if frac_bits is None else frac_bits
        if model == "lif":
            v_all = inputs.lif_v0(n, init_seed) if v0 is None else v0
            st["v"] = torch.as_tensor(v_all[lo:hi]).to(device).contiguous()
            st["ref"] = torch.zeros(n_local, dtype=torch.uint8, device=device)
        else:
            v, m, h, nk = inputs.hh_init(n, init_seed) if v0 is None else v0
            for k, a in (("v", v), ("m", m), ("h", h), ("n", nk)):
                st[k] = torch.as_tensor(a[lo:hi]).to(device).contiguous()
        self.state = st
        # bit-packed spike vector (int32 storage of the uint32 words); a
        # caller may share one vector between partitions on one device
        words = self.part.padded_words if world > 1 else (n + 31) // 32
        self.spikes = (torch.zeros(words, dtype=torch.int32, device=device)
                       if spikes is None else spikes)
        if projections is None:
            # Listing S3: E rows [0, n_exc) -> g_E with w_E, I rows -> g_I with w_I
            if conn == "jit":
                projections = [ProjSpec(0, self.n_exc, "exc", w_exc, seed=seed_e, p=self.p),
                               ProjSpec(self.n_exc, n, "inh", w_inh, seed=seed_i, p=self.p)]
            else:
                (ip_e, ix_e), (ip_i, ix_i) = csr
                projections = [ProjSpec(0, self.n_exc, "exc", w_exc, csr=(ip_e, ix_e)),
                               ProjSpec(self.n_exc, n, "inh", w_inh, csr=(ip_i, ix_i))]
        self.projections = projections
        descs, keep = [], []
        for ps in projections:
            rec = B.RECEPTOR_EXC if ps.receptor == "exc" else B.RECEPTOR_INH
            if ps.csr is None:
                pp = self.p if ps.p is None else ps.p
                jit = B.jitconn_spec(ps.seed, pp, B.conn_len(pp), seg_len)
                descs.append(B.projection(pre_begin=ps.pre_begin, pre_end=ps.pre_end,
                                          weight=ps.weight, receptor=rec, jit=jit))
            else:
                ip, ix, _ = _slice_csr(ps.csr[0], ps.csr[1], lo, hi, device)
                keep += [ip, ix]
                descs.append(B.projection(pre_begin=ps.pre_begin, pre_end=ps.pre_end,
                                          weight=ps.weight, receptor=rec, csr=(ip, ix)))
        self.exchange = exchange
        kw = {}
        if exchange == "nccl":
            nccl_id = share_nccl_id(rank, world, group)
            kw = dict(exchange=B.EXCHANGE_NCCL, rank=rank, world=world,
                      part_len=self.part.local, nccl_id=nccl_id)
        elif exchange != "caller":
            raise ValueError(f"exchange={exchange!r}")
        self.net = B.Network(model=B.MODEL_LIF if model == "lif" else B.MODEL_HH,
                             n=n, state=st, spikes=self.spikes, params=params,
                             projections=descs, col_begin=lo, col_end=hi, delay=delay,
                             keep=keep, **kw)
        self.delay = delay
        self._send = None

    # single device, or the library's NCCL exchange: the whole loop runs in
    # the library
    def run(self, n_steps: int, raster: torch.Tensor | None = None, counts=None):
        self.net.step(n_steps, raster, counts)

    # several devices, caller exchange: scatter -> update -> all-gather, per
    # step.  The all-gather runs on a side stream that waits only for the
    # update kernel's spike words, so it overlaps the local binning kernel
    # (SURVEY 8(e) option (i)); the next scatter waits for it.
    # overlap=False: one stream.
    def step_distributed(self, group=None, raster_row=None, overlap: bool = True):
        if self.exchange == "nccl":
            self.net.step(1, None if raster_row is None else raster_row.view(1, -1))
            return
        if self._send is None:
            self._send = torch.empty(self.part.local_words, dtype=torch.int32,
                                     device=self.spikes.device)
            self._comm = torch.cuda.Stream(device=self.spikes.device)
        self.net.scatter()
        if not overlap:
            self.net.update(raster_row)
            exchange_spikes(self.spikes, self.part, group, self._send)
            return
        compute = torch.cuda.current_stream(self.spikes.device)
        self.net.update_overlap(self._comm, raster_row)
        with torch.cuda.stream(self._comm):
            exchange_spikes(self.spikes, self.part, group, self._send)
        compute.wait_stream(self._comm)

    def capture(self, group=None, overlap: bool = True):
        """CUDA graph of one period of step_distributed -- lcm(2, delay + 1)
        steps, after which the host-side step parity and bucket slot repeat
        -- so a replay costs one launch instead of ~10 host calls per step
        (their enqueue cost is close to the GPU step time).  The exchange is
        captured with it (NCCL; gloo cannot be captured).  Call after at least
        one eager step_distributed; eager steps after the capture put the
        device state out of phase with the graph unless they are a multiple
        of the period.  Returns (graph, steps per replay)."""
        period = math.lcm(2, self.delay + 1)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph):
            for _ in range(period):
                self.step_distributed(group, overlap=overlap)
        return graph, period

    def counters(self):
        return self.net.counters()

    def device_bytes(self) -> int:
        return self.net.device_bytes()


def _slice_csr(indptr, indices, lo, hi, device):
    """Keep the columns [lo, hi) of a row-major CSR, rebased to 0 (8(e))."""
    ip = torch.as_tensor(indptr).to(torch.int64).cpu()
    ix = torch.as_tensor(indices).to(torch.int32).cpu()
    n_rows = ip.numel() - 1
    if lo == 0 and hi >= int(ix.max().item() if ix.numel() else 0) + 1:
        return ip.to(device), ix.to(device), None
    rows = torch.repeat_interleave(torch.arange(n_rows), ip[1:] - ip[:-1])
    keep = (ix >= lo) & (ix < hi)
    rows, cols = rows[keep], ix[keep] - lo
    new_ip = torch.zeros(n_rows + 1, dtype=torch.int64)
    new_ip[1:] = torch.cumsum(torch.bincount(rows, minlength=n_rows), 0)
    return new_ip.to(device), cols.to(torch.int32).contiguous().to(device), None
