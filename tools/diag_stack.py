"""Timing of one stack layer (strided QKV views) vs the contiguous layer at V views."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_08055_b200 as gsa
from paper_2603_08055_b200.stack import GsaStack
V = int(sys.argv[1]) if len(sys.argv) > 1 else 100
L = gsa.build_token_layout(5 * V, V, 36, 36, 4)
p = gsa.GsaParams(window_s=4, top_k=32)
st = GsaStack(L, p, layers=2, heads=16, dim=64, seed=1)
M = L.total_tokens
x = torch.randn(M, 1024, device="cuda").to(torch.bfloat16)
def t(f, n=2):
    f(); torch.cuda.synchronize(); t0 = time.time()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.time() - t0) / n * 1e3
print("gemm ms", t(lambda: x @ st.w_qkv[0]), flush=True)
qkv = x @ st.w_qkv[0]
q, k, v = st.heads_of(qkv)
qc, kc, vc = (a.contiguous() for a in (q, k, v))
out = torch.empty(16, M, 64, device="cuda")
print("layer contiguous ms", t(lambda: gsa.gsa_forward(qc, kc, vc, st.w_g[0], L, p, out=out)), flush=True)
print("layer strided ms", t(lambda: gsa.gsa_forward(q, k, v, st.w_g[0], L, p, out=out)), flush=True)
o2 = torch.empty(M, 16, 64, device="cuda")
print("layer strided + token-major out ms", t(lambda: gsa.gsa_forward(q, k, v, st.w_g[0], L, p, out=o2.permute(1, 0, 2))), flush=True)
print("stack layer ms", t(lambda: st.layer(x, 0)), flush=True)
