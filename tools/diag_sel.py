import sys, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2603_08055_b200 as gsa
from oracle import Layout, Oracle, make_inputs
orc = Oracle()
dev = torch.device("cuda:0")
for lt, H, kk in [((0, 8, 36, 36, 4), 4, 16), ((0, 8, 36, 36, 4), 4, 32), ((0, 8, 36, 36, 4), 16, 16), ((40, 8, 36, 36, 4), 16, 32),
                  ((0, 8, 36, 36, 4), 2, 16), ((0, 8, 36, 36, 4), 4, 8), ((0, 8, 36, 36, 4), 4, 24), ((0, 4, 36, 36, 4), 4, 16)]:
    L = Layout(*lt)
    q, k, v, wg = make_inputs(orc, L, heads=H, dim=64, seed=5)
    tq, tk, tv = (torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in (q, k, v))
    out, ctx = gsa.gsa_forward(tq, tk, tv, torch.from_numpy(wg).to(dev), gsa.build_token_layout(*lt), gsa.GsaParams(window_s=4, top_k=kk), context=True)
    ref = orc.gsa_forward(q, k, v, wg, L, top_k=kk)
    e = (out.cpu() - torch.from_numpy(ref["out"])).abs()
    print(lt, H, kk, 'topk eq', np.array_equal(ctx.topk.cpu().numpy(), ref["topk"]), 'max err', e.max().item(), 'bad heads', (e.amax(dim=(1,2)) > 1e-3).nonzero().flatten().tolist())
