"""Two processes on ONE GPU, gloo process group, the real sm_100a kernels: the
view-sharded layer (ShardedLayer, dist.py) against the unsharded gsa_forward.
usage: torchrun --nproc-per-node 2 --master-addr 127.0.0.1 tools/diag_shard_mp.py"""
import os
import sys

import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2603_08055_b200 as gsa  # noqa: E402
from paper_2603_08055_b200 import dist as gdist  # noqa: E402

rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
torch.cuda.set_device(0)
dist.init_process_group("gloo")
lt = (8 * world, 4 * world, 36, 36, 4)
L = gsa.build_token_layout(*lt)
H, d = 4, 64
g = torch.Generator(device="cuda").manual_seed(11)
q, k, v = (torch.randn(H, L.total_tokens, d, generator=g, device="cuda").to(torch.bfloat16) for _ in range(3))
wg = torch.randn(H, d, d, generator=g, device="cuda") / 8
for variant in (0, 1):
    p = gsa.GsaParams(window_s=4, top_k=16, variant=variant, ref_stride=3)
    ref_out, ctx = gsa.gsa_forward(q, k, v, wg, L, p, context=True)
    spec = gdist.shard_spec(L, rank, world)
    layer = gdist.ShardedLayer(L, p, H, d, rank, world, device="cuda")
    q_own = gdist.own_rows_of(q, L, spec).contiguous()
    k_all = torch.zeros_like(k)
    v_all = torch.zeros_like(v)
    gdist.scatter_own_rows(k_all, gdist.own_rows_of(k, L, spec), L, spec)
    gdist.scatter_own_rows(v_all, gdist.own_rows_of(v, L, spec), L, spec)
    out_own = layer.forward(q_own, k_all, v_all, wg)
    torch.cuda.synchronize()
    exp_own = gdist.own_rows_of(ref_out, L, spec)
    w0, w1 = spec.windows(L)
    ok_topk = torch.equal(layer.ctx_topk, ctx.topk[:, w0:w1])
    ok_kv = torch.equal(k_all, k) and torch.equal(v_all, v)
    err = (out_own - exp_own).abs().max().item()
    print(f"rank {rank} variant {variant}: topk bit-exact {ok_topk}, gathered K/V exact {ok_kv}, max|dout| {err:.2e}",
          flush=True)
    assert ok_topk and ok_kv and err < 1e-5
dist.destroy_process_group()
