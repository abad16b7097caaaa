"""Query-view sharding (paper_2603_08055_b200.dist).

CPU (world_size 2, gloo): the sharded orchestration — shard geometry, own-row
offsets, in-place all-gathers of Kc/Vc and K/V rows, global window ids — runs
with the compute steps replaced by a stand-in built on the oracle, and every
rank's rows must equal the unsharded oracle layer (top-k bit-exact).

GPU: G virtual shards run the sharded C ABI (gsa_shard_pool / _compress /
_attend) one after another on one device and must reproduce the unsharded
sm_100a layer: top-k indices bit-exact, outputs to f32 rounding.
"""
from __future__ import annotations

import os
import socket

import numpy as np
import pytest
import torch

from conftest import ROOT, rel_l2  # noqa: F401
from oracle import Layout, Oracle, make_inputs

import paper_2603_08055_b200 as gsa
from paper_2603_08055_b200 import dist as gdist


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


# ------------------------------------------------------------- shard geometry
def test_shard_spec_partitions_views_and_specials():
    L = gsa.TokenLayout(40, 8, 8, 8, 4)
    specs = [gdist.shard_spec(L, r, 4) for r in range(4)]
    assert [(s.frame_begin, s.frame_end) for s in specs] == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert [(s.special_begin, s.special_end) for s in specs] == [(0, 10), (10, 20), (20, 30), (30, 40)]
    assert specs[1].windows(L) == (2 * 4, 4 * 4)
    assert specs[3].image_rows(L) == (6 * 64, 8 * 64)
    assert sum(s.own_rows(L) for s in specs) == L.total_tokens


def test_shard_spec_rejects_uneven():
    with pytest.raises(gsa.ShapeMismatch):
        gdist.shard_spec(gsa.TokenLayout(5, 3, 8, 8, 4), 0, 2)
    with pytest.raises(gsa.ShapeMismatch):
        gdist.shard_spec(gsa.TokenLayout(4, 4, 8, 8, 4), 2, 2)


def test_own_rows_roundtrip():
    L = gsa.TokenLayout(6, 4, 4, 4, 2)
    x = torch.arange(2 * L.total_tokens * 3, dtype=torch.float32).reshape(2, L.total_tokens, 3)
    y = torch.zeros_like(x)
    for r in range(2):
        spec = gdist.shard_spec(L, r, 2)
        own = gdist.own_rows_of(x, L, spec)
        assert own.shape[1] == spec.own_rows(L)
        gdist.scatter_own_rows(y, own, L, spec)
    assert torch.equal(x, y)


# ---------------------------------------------------- oracle stand-in compute
class OracleOps:
    """The three sharded compute steps on the CPU, from the oracle's row-subset
    entry points (test-only: checks the sharding logic, not the kernels)."""

    def __init__(self, orc: Oracle, lt, params: gsa.GsaParams, spec: gdist.ShardSpec):
        self.orc, self.L, self.p, self.spec = orc, Layout(*lt), params, spec
        self.lt = lt
        self.scale = 1.0 / 8.0

    def _own_windows(self, H):
        w0, w1 = self.spec.frame_begin * self.L.windows_per_frame, self.spec.frame_end * self.L.windows_per_frame
        W = self.L.num_windows
        return w0, w1, np.array([h * W + w for h in range(H) for w in range(w0, w1)], np.int64)

    def pool(self, q_own, k_all, v_all, qc_own, kc_all, vc_all):
        L, s = self.L, self.spec
        ms_g = s.special_end - s.special_begin
        nf = s.frame_end - s.frame_begin
        Lg = Layout(0, nf, L.grid_h, L.grid_w, L.window_s)
        i0, i1 = s.frame_begin * L.tokens_per_frame, s.frame_end * L.tokens_per_frame
        qc_own[:] = torch.from_numpy(self.orc.pool(q_own[:, ms_g:].numpy(), Lg))
        w0, w1, _ = self._own_windows(q_own.shape[0])
        kc_all[:, w0:w1] = torch.from_numpy(self.orc.pool(k_all[:, L.num_special + i0:L.num_special + i1].numpy(), Lg))
        vc_all[:, w0:w1] = torch.from_numpy(self.orc.pool(v_all[:, L.num_special + i0:L.num_special + i1].numpy(), Lg))

    def _excluded(self):
        if self.p.variant != gsa.HYBRID:
            return None
        ex = np.zeros(self.L.num_windows, np.uint8)
        ex[self.orc.forced_windows(self.L, self.p.ref_stride)] = 1
        return ex

    def compress(self, qc_own, kc_all, vc_all, o_comp_own, lse_own, topk_own):
        H, W = kc_all.shape[0], self.L.num_windows
        w0, w1, rows = self._own_windows(H)
        qc_full = np.zeros(kc_all.shape, np.float32)
        qc_full[:, w0:w1] = qc_own.numpy()
        out, lse, idx = self.orc.compress_topk(qc_full, kc_all.numpy(), vc_all.numpy(), self.p.top_k, self.scale,
                                               excluded=self._excluded(), rows=rows)
        ke = idx.shape[1]
        o_comp_own[:] = torch.from_numpy(out.reshape(H, w1 - w0, -1))
        lse_own[:] = torch.from_numpy(lse.reshape(H, w1 - w0))
        topk_own[:, :, :ke] = torch.from_numpy(idx.reshape(H, w1 - w0, ke))
        return ke

    def attend(self, q_own, k_all, v_all, w_g, o_comp_own, topk_own, out_own):
        L, s, orc = self.L, self.spec, self.orc
        H, d = q_own.shape[0], q_own.shape[2]
        ms_g = s.special_end - s.special_begin
        if ms_g:
            o, _ = orc.dense_attention(q_own[:, :ms_g].numpy(), k_all.numpy(), v_all.numpy(), self.scale)
            out_own[:, :ms_g] = torch.from_numpy(o)
        w0, w1, rows = self._own_windows(H)
        W, Ms = L.num_windows, L.num_special
        ke = topk_own.shape[2]
        topk_full = np.zeros((H, W, ke), np.int32)
        topk_full[:, w0:w1] = topk_own.numpy()
        offs, ids = orc.build_plan(topk_full, L, self.p.variant, self.p.ref_stride)
        i0, i1 = s.frame_begin * L.tokens_per_frame, s.frame_end * L.tokens_per_frame
        q_img = np.zeros((H, L.image_tokens, d), np.float32)
        q_img[:, i0:i1] = q_own[:, ms_g:].numpy()
        o_sel, _ = orc.block_sparse(q_img, k_all[:, Ms:].numpy(), v_all[:, Ms:].numpy(), L, offs, ids, self.scale,
                                    rows=rows)
        g = orc.gate(q_own[:, ms_g:].numpy(), w_g.numpy())
        o_sel = o_sel.reshape(H, w1 - w0, -1, d)
        comp = o_comp_own.numpy()
        img = np.empty((H, i1 - i0, d), np.float32)
        for wl in range(w1 - w0):
            toks = np.array(L.tokens_of_window(w0 + wl)) - i0
            gg = g[:, toks]
            img[:, toks] = gg * comp[:, wl][:, None, :] + (np.float32(1) - gg) * o_sel[:, wl]
        out_own[:, ms_g:] = torch.from_numpy(img)


def _gloo_worker(rank, world, port, lt, top_k, variant, result_q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        orc = Oracle()
        L = Layout(*lt)
        q, k, v, wg = make_inputs(orc, L, heads=2, dim=64, seed=11)
        layout = gsa.TokenLayout(*lt)
        params = gsa.GsaParams(window_s=lt[4], top_k=top_k, variant=variant, ref_stride=2)
        spec = gdist.shard_spec(layout, rank, world)
        tq, tk, tv = (torch.from_numpy(x) for x in (q, k, v))
        q_own = gdist.own_rows_of(tq, layout, spec)
        # only the rank's own K/V rows are present before the gather
        k_all, v_all = torch.full_like(tk, float("nan")), torch.full_like(tv, float("nan"))
        gdist.scatter_own_rows(k_all, gdist.own_rows_of(tk, layout, spec), layout, spec)
        gdist.scatter_own_rows(v_all, gdist.own_rows_of(tv, layout, spec), layout, spec)
        layer = gdist.ShardedLayer(layout, params, 2, 64, rank, world, device="cpu",
                                   ops=OracleOps(orc, lt, params, spec))
        out_own = layer.forward(q_own, k_all, v_all, torch.from_numpy(wg))
        ok_kv = bool(torch.equal(k_all, tk) and torch.equal(v_all, tv))
        result_q.put((rank, out_own.numpy(), layer.ctx_topk.numpy().copy(), ok_kv))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("lt,top_k,variant", [((4, 4, 8, 8, 4), 5, 0), ((2, 4, 8, 8, 4), 6, 1),
                                              ((0, 2, 8, 12, 2), 9, 0)])
def test_sharded_layer_gloo_world2_matches_unsharded(orc, lt, top_k, variant):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q_ = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gloo_worker, args=(r, 2, port, lt, top_k, variant, q_)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        r, out, topk, ok_kv = q_.get(timeout=300)
        res[r] = (out, topk, ok_kv)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    L = Layout(*lt)
    q, k, v, wg = make_inputs(orc, L, heads=2, dim=64, seed=11)
    ref = orc.gsa_forward(q, k, v, wg, L, top_k=top_k, variant=variant, ref_stride=2)
    layout = gsa.TokenLayout(*lt)
    full = torch.zeros(2, L.total_tokens, 64)
    for r in range(2):
        out, topk, ok_kv = res[r]
        assert ok_kv, "the in-place all-gather did not complete K/V"
        spec = gdist.shard_spec(layout, r, 2)
        w0, w1 = spec.windows(layout)
        np.testing.assert_array_equal(topk, ref["topk"][:, w0:w1])
        gdist.scatter_own_rows(full, torch.from_numpy(out), layout, spec)
    np.testing.assert_allclose(full.numpy(), ref["out"], rtol=0, atol=1e-6)


# ------------------------------------------------------- GPU: virtual shards
@pytest.mark.gpu
@pytest.mark.parametrize("G,lt,variant", [(2, (10, 2, 16, 16, 4), 0), (4, (40, 8, 36, 36, 4), 0),
                                          (4, (20, 8, 16, 16, 4), 1), (5, (0, 10, 16, 16, 4), 0)])
def test_virtual_shards_match_unsharded_gpu(G, lt, variant):
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    orc = Oracle()
    L = Layout(*lt)
    q, k, v, wg = make_inputs(orc, L, heads=4, dim=64, seed=5)
    dev = torch.device("cuda:0")
    tq, tk, tv = (torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in (q, k, v))
    twg = torch.from_numpy(wg).to(dev)
    layout = gsa.build_token_layout(*lt)
    params = gsa.GsaParams(window_s=lt[4], top_k=16, variant=variant, ref_stride=3)
    full_out, ctx = gsa.gsa_forward(tq, tk, tv, twg, layout, params, context=True)
    H, W, d = 4, layout.num_windows, 64
    kc_all = torch.empty(H, W, d, device=dev)
    vc_all = torch.empty(H, W, d, device=dev)
    shards = []
    for r in range(G):
        spec = gdist.shard_spec(layout, r, G)
        ops = gdist.DeviceOps(layout, params, spec, H, d, dev)
        q_own = gdist.own_rows_of(tq, layout, spec).contiguous()
        w0, w1 = spec.windows(layout)
        qc_own = torch.empty(H, w1 - w0, d, device=dev)
        ops.pool(q_own, tk, tv, qc_own, kc_all, vc_all)
        shards.append((spec, ops, q_own, qc_own, w0, w1))
    torch.cuda.synchronize()
    assert torch.equal(kc_all, ctx.kc) and torch.equal(vc_all, ctx.vc), "sharded pooling is not bit-exact"
    got = torch.zeros_like(full_out)
    for spec, ops, q_own, qc_own, w0, w1 in shards:
        o_comp = torch.empty(H, w1 - w0, d, device=dev)
        lse = torch.empty(H, w1 - w0, device=dev)
        topk = torch.empty(H, w1 - w0, ctx.k_eff, dtype=torch.int32, device=dev)
        ke = ops.compress(qc_own, kc_all, vc_all, o_comp, lse, topk)
        assert ke == ctx.k_eff
        assert torch.equal(topk, ctx.topk[:, w0:w1]), "sharded top-k differs from the unsharded layer"
        out_own = torch.empty(H, spec.own_rows(layout), d, device=dev)
        ops.attend(q_own, tk, tv, twg, o_comp, topk, out_own)
        gdist.scatter_own_rows(got, out_own, layout, spec)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(ctx.topk.cpu().numpy(), orc.gsa_forward(q, k, v, wg, L, top_k=16, variant=variant,
                                                                         ref_stride=3)["topk"])
    assert (got - full_out).abs().max().item() < 1e-5


@pytest.mark.gpu
def test_sharded_layer_two_processes_one_gpu():
    """The view-sharded layer across two real processes (torchrun, gloo group, both on
    cuda:0, the sm_100a kernels): gathered K/V exact, top-k bit-exact and outputs equal
    to the unsharded gsa_forward, plain and hybrid (tools/diag_shard_mp.py)."""
    import subprocess
    import sys

    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", "29547",
                        os.path.join(root, "tools", "diag_shard_mp.py")],
                       capture_output=True, text=True, timeout=600, cwd=root)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count("topk bit-exact True, gathered K/V exact True") == 4, r.stdout


def test_shard_of_rank_and_gather_plan_cover_every_row():
    """The C plan (gsa_shard_gather_plan) run by both gsa_shard_forward (NCCL) and the
    torch.distributed path: over all ranks its blocks tile every Kc/Vc row and every K/V
    row of every head exactly once, and gsa_shard_of_rank matches the equal-block split."""
    import paper_2603_08055_b200 as gsa
    from paper_2603_08055_b200.dist import gather_plan, shard_spec
    for lt, world in (((40, 8, 36, 36, 4), 4), ((0, 6, 8, 12, 4), 3), ((6, 2, 8, 8, 2), 2), ((5, 5, 4, 4, 4), 5)):
        L = gsa.build_token_layout(*lt)
        H, d = 3, 64
        M, W = L.total_tokens, L.num_windows
        for r in range(world):
            s = shard_spec(L, r, world)
            assert (s.frame_begin, s.frame_end) == (r * lt[1] // world, (r + 1) * lt[1] // world)
            assert (s.special_begin, s.special_end) == (r * lt[0] // world, (r + 1) * lt[0] // world)
        kv_hs = M * d + 64  # a padded head stride is allowed
        plan = gather_plan(L, world, H, d, kv_hs)
        cover = {0: np.zeros(H * W * d, np.int32), 1: np.zeros(H * W * d, np.int32),
                 2: np.zeros(H * kv_hs, np.int32), 3: np.zeros(H * kv_hs, np.int32)}
        for b, phase, off, cnt in plan:
            assert phase == (0 if b < 2 else 1)
            cover[b][off:off + world * cnt] += 1
        for b in (0, 1):
            assert (cover[b] == 1).all()
        for b in (2, 3):
            c = cover[b].reshape(H, kv_hs)
            assert (c[:, :M * d] == 1).all() and (c[:, M * d:] == 0).all()
    with pytest.raises(gsa.ShapeMismatch):
        shard_spec(gsa.build_token_layout(5, 5, 4, 4, 4), 0, 2)


def test_comm_init_fails_cleanly_without_a_gpu():
    """gsa_comm_* report status codes (NcclError / CudaError), never crash, when the
    process has no usable GPU (this CPU box)."""
    import ctypes as C
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("needs a GPU-less process")
    from paper_2603_08055_b200 import _lib
    L = _lib.load()
    comm = C.c_void_p()
    rc = L.gsa_comm_init(C.byref(comm), (C.c_char * 128)(), 1, 0)
    assert rc in (11, 13), rc  # GSA_ERR_CUDA / GSA_ERR_NCCL
    assert L.gsa_comm_destroy(None) == 0


@pytest.mark.gpu
@pytest.mark.parametrize("variant", [0, 1])
def test_nccl_sharded_layer_single_rank_matches_forward(variant):
    """gsa_shard_forward through a real NCCL communicator (one rank: the only GPU this
    box has) equals gsa_forward: top-k bit-exact, output to f32 rounding."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2603_08055_b200 as gsa
    from paper_2603_08055_b200.dist import NcclShardedLayer
    lt = (40, 8, 36, 36, 4)
    L = gsa.build_token_layout(*lt)
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k, v = (torch.randn(4, L.total_tokens, 64, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
    wg = torch.randn(4, 64, 64, generator=g, device="cuda") / 8
    p = gsa.GsaParams(window_s=4, top_k=16, variant=variant, ref_stride=3)
    ref, ctx = gsa.gsa_forward(q, k, v, wg, L, p, context=True)
    layer = NcclShardedLayer(L, p, 4, 64, 0, 1)
    out = layer.forward(q, k.clone(), v.clone(), wg)
    torch.cuda.synchronize()
    assert torch.equal(layer.ctx_topk, ctx.topk)
    assert float((out - ref).abs().max()) < 1e-5
    layer.close()
