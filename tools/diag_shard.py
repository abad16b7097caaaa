import sys, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2603_08055_b200 as gsa
from paper_2603_08055_b200 import dist as gdist
from oracle import Layout, Oracle, make_inputs
orc = Oracle()
for G, lt in [(4, (40, 8, 36, 36, 4)), (2, (40, 8, 36, 36, 4)), (4, (0, 8, 36, 36, 4)), (4, (40, 8, 16, 16, 4))]:
    L = Layout(*lt)
    q, k, v, wg = make_inputs(orc, L, heads=4, dim=64, seed=5)
    dev = torch.device("cuda:0")
    tq, tk, tv = (torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in (q, k, v))
    twg = torch.from_numpy(wg).to(dev)
    layout = gsa.build_token_layout(*lt)
    params = gsa.GsaParams(window_s=4, top_k=16)
    full_out, ctx = gsa.gsa_forward(tq, tk, tv, twg, layout, params, context=True)
    H, W, d = 4, layout.num_windows, 64
    kc_all = torch.empty(H, W, d, device=dev); vc_all = torch.empty(H, W, d, device=dev)
    got = torch.zeros_like(full_out)
    specs = [gdist.shard_spec(layout, r, G) for r in range(G)]
    opss = [gdist.DeviceOps(layout, params, s, H, d, dev) for s in specs]
    qowns = [gdist.own_rows_of(tq, layout, s).contiguous() for s in specs]
    qcs = []
    for s, ops, qo in zip(specs, opss, qowns):
        w0, w1 = s.windows(layout); qc = torch.empty(H, w1 - w0, d, device=dev); ops.pool(qo, tk, tv, qc, kc_all, vc_all); qcs.append(qc)
    for s, ops, qo, qc in zip(specs, opss, qowns, qcs):
        w0, w1 = s.windows(layout)
        oc = torch.empty(H, w1 - w0, d, device=dev); lse = torch.empty(H, w1 - w0, device=dev)
        tk_ = torch.empty(H, w1 - w0, ctx.k_eff, dtype=torch.int32, device=dev)
        ops.compress(qc, kc_all, vc_all, oc, lse, tk_)
        print(' oc err', (oc - ctx.o_comp_coarse[:, w0:w1]).abs().max().item(), 'topk eq', torch.equal(tk_, ctx.topk[:, w0:w1]))
        oo = torch.empty(H, s.own_rows(layout), d, device=dev)
        ops.attend(qo, tk, tv, twg, oc, tk_, oo)
        gdist.scatter_own_rows(got, oo, layout, s)
    torch.cuda.synchronize()
    e = (got - full_out).abs()
    Ms = lt[0]
    print(G, lt, 'special err', e[:, :Ms].max().item() if Ms else 0, 'image err', e[:, Ms:].max().item())
    per_frame = e[:, Ms:].reshape(H, lt[1], -1, d).amax(dim=(0, 2, 3))
    print('  per frame', [round(x, 4) for x in per_frame.tolist()])
