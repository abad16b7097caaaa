"""Selection-kernel locality probe: the same layer with (a) random Q/K (iid
selections, gathers from HBM) and (b) every query window selecting the same 32
key windows (gathers hit L2). If (b) is much faster the kernel is memory-bound."""
import sys, torch, json
sys.path.insert(0, '.')
import paper_2603_08055_b200 as gsa
from paper_2603_08055_b200 import _lib
import ctypes
V = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
L = gsa.build_token_layout(5 * V, V, 36, 36, 4)
M = L.total_tokens
dev = torch.device('cuda:0')
g = torch.Generator(device=dev).manual_seed(1)
q, k, v = (torch.randn(16, M, 64, generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
wg = torch.randn(16, 64, 64, generator=g, device=dev) / 8
p = gsa.GsaParams(window_s=4, top_k=32)
lib = _lib.load()
def timed(q, k, v, reps=3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    for e in ev: e.record()
    h = (ctypes.c_void_p * 5)(*[e.cuda_event for e in ev])
    gsa.gsa_forward(q, k, v, wg, L, p)
    torch.cuda.synchronize()
    out = []
    for _ in range(reps):
        lib.gsa_set_stage_events(h, 5)
        gsa.gsa_forward(q, k, v, wg, L, p)
        lib.gsa_set_stage_events(None, 0)
        torch.cuda.synchronize()
        out.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
    return min(out, key=lambda r: r[3])
print('random   special/pool/compress/select ms', [round(x, 2) for x in timed(q, k, v)])
q2 = torch.ones_like(q) * 0.5 + 0.01 * q.float().to(torch.bfloat16)
k2 = k.clone()
ms = L.num_special
for w in range(32):
    for t in L.tokens_of_window(w) if hasattr(L, 'tokens_of_window') else []:
        k2[:, ms + t] = 4.0
print('same-32  special/pool/compress/select ms', [round(x, 2) for x in timed(q2.to(torch.bfloat16), k2, v)])
