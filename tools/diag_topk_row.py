import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_2603_08055_b200 as gsa
sys.path.insert(0, 'tools')
V = 1000
ns, nf, gh, gw, s = 5 * V, V, 36, 36, 4
dev = torch.device('cuda:0')
gen = torch.Generator(device=dev).manual_seed(7)
M = ns + nf * gh * gw
q, k, v = (torch.randn(16, M, 64, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16) for _ in range(3))
L = gsa.build_token_layout(ns, nf, gh, gw, s)
qc = gsa.avg_pool_tokens(q[:1, ns:], L)[0]
kc = gsa.avg_pool_tokens(k[:1, ns:], L)[0]
def sim(x, K=32, nb=8):
    W = x.size
    t0 = np.sort(x[:128])[::-1]; LB = t0[K-1]; mx = t0[0]; span = mx - LB
    delta = span / nb if span > 0 else abs(LB) / 1024
    cnt = np.zeros(nb, int); cands = 0; hist = []
    for t in range(0, W, 128):
        tile = x[t:t+128]; c = tile[tile >= LB]; cands += c.size
        for v_ in c: cnt[min(nb-1, int((v_ - LB) / delta))] += 1
        suf = np.cumsum(cnt[::-1])[::-1]
        js = [j for j in range(1, nb) if suf[j] >= K]
        if js:
            j = max(js); LB += j * delta; cnt = np.concatenate([cnt[j:], np.zeros(j, int)])
            if j == nb - 1:
                c2 = np.zeros(nb, int); c2[:4] = cnt[0::2] + cnt[1::2]; cnt = c2; delta *= 2
        if t // 128 in (0, 1, 2, 5, 10, 50, 200, 600): hist.append((t // 128, round(float(LB), 4), round(float(delta), 5), cands))
    return cands, hist
for w in [1255, 28696, 5, 100]:
    x = (qc[w:w+1] @ kc.T)[0].cpu().numpy()
    c, hst = sim(x)
    srt = np.sort(x)[::-1]
    print('row', w, 'cands', c, 'tau', srt[31], 'max', srt[0], 'tile0 top:', np.sort(x[:128])[::-1][:4], np.sort(x[:128])[::-1][31])
    print('   ', hst)
