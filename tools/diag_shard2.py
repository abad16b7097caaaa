import sys, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2603_08055_b200 as gsa
from paper_2603_08055_b200 import dist as gdist
from oracle import Layout, Oracle, make_inputs
orc = Oracle()
G, lt = 4, (0, 8, 36, 36, 4)
L = Layout(*lt)
q, k, v, wg = make_inputs(orc, L, heads=4, dim=64, seed=5)
dev = torch.device("cuda:0")
tq, tk, tv = (torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in (q, k, v))
twg = torch.from_numpy(wg).to(dev)
layout = gsa.build_token_layout(*lt)
params = gsa.GsaParams(window_s=4, top_k=16)
full_out, ctx = gsa.gsa_forward(tq, tk, tv, twg, layout, params, context=True)
H, W, d = 4, layout.num_windows, 64
for r in [0, 2]:
    s = gdist.shard_spec(layout, r, G)
    ops = gdist.DeviceOps(layout, params, s, H, d, dev)
    w0, w1 = s.windows(layout)
    qo = gdist.own_rows_of(tq, layout, s).contiguous()
    oc = ctx.o_comp_coarse[:, w0:w1].contiguous()
    tk_ = ctx.topk[:, w0:w1].contiguous()
    oo = torch.empty(H, s.own_rows(layout), d, device=dev)
    ops.attend(qo, tk, tv, twg, oc, tk_, oo)
    torch.cuda.synchronize()
    i0, i1 = s.image_rows(layout)
    e = (oo - full_out[:, i0:i1]).abs().amax(dim=2)  # [H][tokens]
    print('shard', r, 'max err', e.max().item())
    bad = (e > 1e-5).nonzero()
    print(' bad count', bad.shape[0], 'of', e.numel())
    if bad.shape[0]:
        toks = bad[:, 1].unique()
        print(' heads', bad[:, 0].unique().tolist(), 'first toks', toks[:20].tolist(), 'last', toks[-5:].tolist())
        # window of token
        wins = sorted(set(layout.window_of_token(int(t)) for t in toks.tolist()))
        print(' bad local windows', len(wins), wins[:20], wins[-5:])
ref = orc.gsa_forward(q, k, v, wg, L, top_k=16)
ro = torch.from_numpy(ref["out"]).to(dev)
print('unsharded vs oracle', (full_out - ro).abs().max().item())
s = gdist.shard_spec(layout, 2, G); i0, i1 = s.image_rows(layout)
print('topk eq oracle', np.array_equal(ctx.topk.cpu().numpy(), ref["topk"]))
