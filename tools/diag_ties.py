"""Near-tie stress: K/V tokens = a shared vector + eps * noise (over-smoothed
activations). Times gsa_forward at V views and prints the compress candidate
statistics (GSA_DEBUG_STATS=1 in the environment)."""
import sys, time
import torch
sys.path.insert(0, ".")
import paper_2603_08055_b200 as gsa
V = int(sys.argv[1]) if len(sys.argv) > 1 else 100
L = gsa.build_token_layout(5 * V, V, 36, 36, 4)
p = gsa.GsaParams(window_s=4, top_k=32)
M = L.total_tokens
g = torch.Generator(device="cuda").manual_seed(1)
q = torch.randn(16, M, 64, generator=g, device="cuda").to(torch.bfloat16)
base = torch.randn(16, 1, 64, generator=g, device="cuda")
wg = torch.randn(16, 64, 64, generator=g, device="cuda") / 8
for eps in [float(e) for e in (sys.argv[2:] or ["1", "0.1", "0.01", "0.001"])]:
    k = (base + eps * torch.randn(16, M, 64, generator=g, device="cuda")).to(torch.bfloat16)
    v = torch.randn(16, M, 64, generator=g, device="cuda").to(torch.bfloat16)
    torch.cuda.synchronize(); t0 = time.time()
    out = gsa.gsa_forward(q, k, v, wg, L, p)
    torch.cuda.synchronize()
    print(f"eps {eps}: {1e3 * (time.time() - t0):.1f} ms", flush=True)
