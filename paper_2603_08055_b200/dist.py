"""Query-view sharding of one GSA layer over G GPUs (one process per GPU).

The reference is a single-process CPU library (no comms); this is
the multi-GPU partition BASELINE.json's north star asks for, built on the
sharded C ABI (include/gsa_sm100.h, gsa_shard_*). Rank g owns a contiguous
block of views (frames) and the matching block of special rows:

    frames   [g*V/G, (g+1)*V/G)        -> its query windows and image rows
    specials [g*Ms/G, (g+1)*Ms/G)      -> its dense special-token rows

Every (head, query-window) row of the compressed branch and every query of
the selection branch is independent given ALL pooled keys Kc/Vc and ALL K/V
rows, so one layer is

    1. pool own Q/K/V windows           (gsa_shard_pool; K/V windows land at
                                         their global rows of kc_all / vc_all)
    2. all-gather Kc, Vc  (f32)         -- gates step 3
       all-gather K, V rows (bf16)      -- issued right after, runs on NCCL's
                                           stream concurrently with step 3
    3. compressed attention + top-k of own windows vs all W windows
                                        (gsa_shard_compress; global window ids)
    4. own specials over all M keys, own windows' selection + gate + merge
                                        (gsa_shard_attend)

Qc, top-k indices and outputs never leave the rank. Buffers are head-major
[H][rows][d] like the reference's Tensor<T>, so a rank's rows are contiguous
per head and the gathers are per-head all_gather_into_tensor calls, coalesced
into one NCCL group where the backend supports it (gloo, used by the CPU
tests, does not).

The compute steps are pluggable (`ops`): DeviceOps calls the sm_100a library;
the CPU tests substitute a stand-in built on the oracle to check the sharding
logic (index math, offsets, collectives) with world_size 2 over gloo.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import torch
import torch.distributed as dist

from .gsa import GsaParams, ShapeMismatch, TokenLayout, _check, _desc, _ptr, _stream
from . import _lib


@dataclass(frozen=True)
class ShardSpec:
    """A rank's share of the layout (mirrors gsa_shard in include/gsa_sm100.h)."""
    frame_begin: int
    frame_end: int
    special_begin: int
    special_end: int

    def c(self):
        return _lib.GsaShard(self.frame_begin, self.frame_end, self.special_begin, self.special_end)

    def windows(self, layout: TokenLayout) -> tuple[int, int]:
        return self.frame_begin * layout.windows_per_frame, self.frame_end * layout.windows_per_frame

    def image_rows(self, layout: TokenLayout) -> tuple[int, int]:
        return self.frame_begin * layout.tokens_per_frame, self.frame_end * layout.tokens_per_frame

    def own_rows(self, layout: TokenLayout) -> int:
        return (self.special_end - self.special_begin) + (self.frame_end - self.frame_begin) * layout.tokens_per_frame


def shard_spec(layout: TokenLayout, rank: int, world: int) -> ShardSpec:
    """Contiguous equal blocks of views and specials (gsa_shard_of_rank). Equal blocks
    keep every all-gather a plain ncclAllGather (equal counts), so the view and special
    counts must divide by the world size."""
    if world < 1 or not 0 <= rank < world:
        raise ShapeMismatch(f"rank {rank} outside world {world}")
    out = _lib.GsaShard()
    _check(_lib.load().gsa_shard_of_rank(C.byref(layout.c()), world, rank, C.byref(out)))
    return ShardSpec(out.frame_begin, out.frame_end, out.special_begin, out.special_end)


def gather_plan(layout: TokenLayout, world: int, heads: int, dim: int, kv_head_stride: int):
    """The in-place all-gathers of one sharded layer (gsa_shard_gather_plan; identical on
    every rank): [(buffer, phase, offset, count)], buffer 0/1 = kc_all/vc_all, 2/3 =
    k_all/v_all (flat element offsets; rank r's block at offset + r * count)."""
    L = _lib.load()
    n = C.c_int()
    _check(L.gsa_shard_gather_plan(C.byref(layout.c()), world, heads, dim, kv_head_stride, None, 0, C.byref(n)))
    ops = (_lib.GsaGatherOp * max(1, n.value))()
    _check(L.gsa_shard_gather_plan(C.byref(layout.c()), world, heads, dim, kv_head_stride, ops, n.value,
                                   C.byref(n)))
    return [(o.buffer, o.phase, o.offset, o.count) for o in ops[: n.value]]


def own_rows_of(x: torch.Tensor, layout: TokenLayout, spec: ShardSpec) -> torch.Tensor:
    """The rank's rows of a full [H][M][d] tensor: own specials, then own image rows."""
    i0, i1 = spec.image_rows(layout)
    ms = layout.num_special
    return torch.cat([x[:, spec.special_begin:spec.special_end], x[:, ms + i0:ms + i1]], dim=1)


def scatter_own_rows(full: torch.Tensor, own: torch.Tensor, layout: TokenLayout, spec: ShardSpec) -> None:
    """Inverse of own_rows_of: write a rank's rows into their global positions."""
    i0, i1 = spec.image_rows(layout)
    ms, ns = layout.num_special, spec.special_end - spec.special_begin
    full[:, spec.special_begin:spec.special_end] = own[:, :ns]
    full[:, ms + i0:ms + i1] = own[:, ns:]


# --------------------------------------------------------------- compute ops
class DeviceOps:
    """The sm_100a kernels through the sharded C ABI."""

    def __init__(self, layout: TokenLayout, params: GsaParams, spec: ShardSpec, heads: int, dim: int, device):
        self.L = _lib.load()
        self.lc, self.pc, self.sc = layout.c(), params.c(), spec.c()
        nbytes = self.L.gsa_shard_workspace_bytes(C.byref(self.lc), C.byref(self.pc), C.byref(self.sc), heads, dim)
        if nbytes == 0:
            raise ShapeMismatch("gsa_shard_workspace_bytes rejected the shard / params")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=device)

    def pool(self, q_own, k_all, v_all, qc_own, kc_all, vc_all):
        _check(self.L.gsa_shard_pool(C.byref(_desc(q_own)), C.byref(_desc(k_all)), C.byref(_desc(v_all)),
                                     C.byref(self.lc), C.byref(self.pc), C.byref(self.sc), C.byref(_desc(qc_own)),
                                     C.byref(_desc(kc_all)), C.byref(_desc(vc_all)), _stream()))

    def compress(self, qc_own, kc_all, vc_all, o_comp_own, lse_own, topk_own) -> int:
        ke = C.c_int()
        _check(self.L.gsa_shard_compress(C.byref(_desc(qc_own)), C.byref(_desc(kc_all)), C.byref(_desc(vc_all)),
                                         C.byref(self.lc), C.byref(self.pc), C.byref(self.sc),
                                         C.byref(_desc(o_comp_own)), _ptr(lse_own), _ptr(topk_own), C.byref(ke),
                                         _ptr(self.ws), self.ws.numel(), _stream()))
        return ke.value

    def attend(self, q_own, k_all, v_all, w_g, o_comp_own, topk_own, out_own):
        _check(self.L.gsa_shard_attend(C.byref(_desc(q_own)), C.byref(_desc(k_all)), C.byref(_desc(v_all)),
                                       C.byref(_desc(w_g)), C.byref(self.lc), C.byref(self.pc), C.byref(self.sc),
                                       C.byref(_desc(o_comp_own)), _ptr(topk_own), C.byref(_desc(out_own)),
                                       _ptr(self.ws), self.ws.numel(), _stream()))


# ---------------------------------------------------------------- collectives
def _run_gathers(bufs, plan, phase: int, rank: int, world: int, group, coalesce: bool):
    """In-place all-gathers of the C plan's ops of one phase over flat views of the
    (contiguous) buffers. Returns a handle whose wait() orders the current stream
    after the gathers."""
    calls = []
    for b, ph, off, cnt in plan:
        if ph != phase or cnt == 0:
            continue
        flat = bufs[b].view(-1)
        out = flat[off:off + world * cnt]
        calls.append((out, out[rank * cnt:(rank + 1) * cnt]))
    if coalesce:
        with dist._coalescing_manager(group, calls[0][0].device if calls else None, async_ops=True) as cm:
            for out, inp in calls:
                dist.all_gather_into_tensor(out, inp, group=group)
        return cm
    works = [dist.all_gather_into_tensor(out, inp.clone(), group=group, async_op=True) for out, inp in calls]

    class _All:
        def wait(self):
            for w in works:
                w.wait()
    return _All()


class ShardedLayer:
    """One GSA layer forward, partitioned by query views over a process group.

    forward(q_own, k_all, v_all, w_g) -> out_own
      q_own : [H][Ms_g + Mi_g][d] the rank's query rows (own specials first)
      k_all, v_all : [H][M][d] with the rank's own rows filled in; the other
              ranks' rows are completed in place by the all-gather
      out_own : [H][Ms_g + Mi_g][d] f32, the rank's rows of the unsharded output
    Top-k indices (ctx_topk) are global window ids, bit-exact with gsa_forward.
    """

    def __init__(self, layout: TokenLayout, params: GsaParams, heads: int, dim: int, rank: int, world: int,
                 group=None, device=None, ops=None):
        self.layout, self.params, self.heads, self.dim = layout, params, heads, dim
        self.rank, self.world, self.group = rank, world, group
        self.spec = shard_spec(layout, rank, world)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.ops = ops if ops is not None else DeviceOps(layout, params, self.spec, heads, dim, self.device)
        W = layout.num_windows
        w0, w1 = self.spec.windows(layout)
        self.W_g = w1 - w0
        f = dict(dtype=torch.float32, device=self.device)
        self.kc_all = torch.empty(heads, W, dim, **f)
        self.vc_all = torch.empty(heads, W, dim, **f)
        self.qc_own = torch.empty(heads, self.W_g, dim, **f)
        self.o_comp_own = torch.empty(heads, self.W_g, dim, **f)
        self.lse_own = torch.empty(heads, self.W_g, **f)
        nf = 0
        if params.variant == 1 and params.ref_stride >= 1:
            nf = len(range(0, layout.num_frames, params.ref_stride)) * layout.windows_per_frame
        self.k_eff = max(0, min(params.top_k, W - nf))
        self.topk_own = torch.empty(heads, self.W_g, max(1, self.k_eff), dtype=torch.int32, device=self.device)
        backend = dist.get_backend(group) if world > 1 else None
        self.coalesce = backend == "nccl"
        self.events = None  # optional 4 CUDA events: start, pooled, compressed, done (bench stage times)

    def _mark(self, i):
        if self.events is not None:
            self.events[i].record()

    def forward(self, q_own, k_all, v_all, w_g, out_own: Optional[torch.Tensor] = None):
        L, spec = self.layout, self.spec
        if out_own is None:
            out_own = torch.empty(self.heads, spec.own_rows(L), self.dim, dtype=torch.float32, device=self.device)
        self._mark(0)
        # 1. pooling of own windows (own K/V rows are already in place)
        self.ops.pool(q_own, k_all, v_all, self.qc_own, self.kc_all, self.vc_all)
        self._mark(1)
        if self.world > 1:
            # 2. the C plan's gathers (gsa_shard_gather_plan): Kc/Vc first (gates the
            #    compressed branch), then K/V rows (gates step 4); both queue on the group's
            #    NCCL stream, so the K/V transfer overlaps step 3
            if not (k_all.is_contiguous() and v_all.is_contiguous()):
                raise ShapeMismatch("sharded layer: k_all / v_all must be contiguous [H][M][d]")
            plan = gather_plan(L, self.world, self.heads, self.dim, k_all.stride(0))
            bufs = [self.kc_all, self.vc_all, k_all, v_all]
            h_c = _run_gathers(bufs, plan, 0, self.rank, self.world, self.group, self.coalesce)
            h_kv = _run_gathers(bufs, plan, 1, self.rank, self.world, self.group, self.coalesce)
            h_c.wait()
        # 3. compressed attention + top-k: own query windows vs all windows
        ke = self.ops.compress(self.qc_own, self.kc_all, self.vc_all, self.o_comp_own, self.lse_own, self.topk_own)
        self.k_eff = ke
        self._mark(2)
        if self.world > 1:
            h_kv.wait()
        # 4. own specials (dense over all keys) + own windows' selection, gate, merge
        self.ops.attend(q_own, k_all, v_all, w_g, self.o_comp_own, self.topk_own, out_own)
        self._mark(3)
        return out_own

    @property
    def ctx_topk(self):
        return self.topk_own[:, :, :self.k_eff]


class NcclShardedLayer:
    """The view-sharded layer at the C level: one NCCL communicator (gsa_comm_init,
    libnccl resolved by the library) and gsa_shard_forward, which runs pool -> Kc/Vc
    all-gather -> compress -> selection with the K/V-row all-gather overlapping the
    compressed branch on the communicator's stream (include/gsa_sm100.h). The id is
    exchanged through the caller's torch.distributed group (or passed in)."""

    def __init__(self, layout: TokenLayout, params: GsaParams, heads: int, dim: int, rank: int, world: int,
                 group=None, device=None, unique_id: Optional[bytes] = None):
        self.L = _lib.load()
        self.layout, self.params, self.heads, self.dim = layout, params, heads, dim
        self.rank, self.world = rank, world
        self.spec = shard_spec(layout, rank, world)
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if unique_id is None:
            buf = (C.c_char * 128)()
            if rank == 0:
                _check(self.L.gsa_comm_get_unique_id(buf))
            obj = [bytes(buf)]
            if world > 1:
                dist.broadcast_object_list(obj, src=0, group=group)
            unique_id = obj[0]
        idb = (C.c_char * 128).from_buffer_copy(unique_id)
        self.comm = C.c_void_p()
        with torch.cuda.device(self.device):
            _check(self.L.gsa_comm_init(C.byref(self.comm), idb, world, rank))
        self.lc, self.pc = layout.c(), params.c()
        nbytes = self.L.gsa_shard_forward_workspace_bytes(C.byref(self.lc), C.byref(self.pc), world, rank, heads, dim)
        if nbytes == 0:
            raise ShapeMismatch("gsa_shard_forward_workspace_bytes rejected the layout / params")
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        W = layout.num_windows
        nf = 0
        if params.variant == 1 and params.ref_stride >= 1:
            nf = len(range(0, layout.num_frames, params.ref_stride)) * layout.windows_per_frame
        self.k_eff = max(0, min(params.top_k, W - nf))
        w0, w1 = self.spec.windows(layout)
        self.topk_own = torch.empty(heads, w1 - w0, max(1, self.k_eff), dtype=torch.int32, device=self.device)

    def forward(self, q_own, k_all, v_all, w_g, out_own: Optional[torch.Tensor] = None):
        if out_own is None:
            out_own = torch.empty(self.heads, self.spec.own_rows(self.layout), self.dim, dtype=torch.float32,
                                  device=self.device)
        _check(self.L.gsa_shard_forward(self.comm, C.byref(_desc(q_own)), C.byref(_desc(k_all)),
                                        C.byref(_desc(v_all)), C.byref(_desc(w_g.contiguous())), C.byref(self.lc),
                                        C.byref(self.pc), C.byref(_desc(out_own)), _ptr(self.topk_own),
                                        _ptr(self.ws), self.ws.numel(), _stream()))
        return out_own

    @property
    def ctx_topk(self):
        return self.topk_own[:, :, :self.k_eff]

    def close(self):
        if self.comm:
            _check(self.L.gsa_comm_destroy(self.comm))
            self.comm = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
