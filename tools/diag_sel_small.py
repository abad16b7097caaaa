import sys, torch, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2603_08055_b200 as gsa
from oracle import Layout, Oracle, make_inputs
orc = Oracle()
lt = tuple(int(x) for x in sys.argv[1].split(','))
H, k = int(sys.argv[2]), int(sys.argv[3])
L = Layout(*lt)
q, k_, v, wg = make_inputs(orc, L, heads=H, dim=64, seed=5)
dev = torch.device('cuda:0')
tq, tk, tv = (torch.from_numpy(x).to(dev).to(torch.bfloat16) for x in (q, k_, v))
out = gsa.gsa_forward(tq, tk, tv, torch.from_numpy(wg).to(dev), gsa.build_token_layout(*lt), gsa.GsaParams(window_s=4, top_k=k))
torch.cuda.synchronize()
ref = orc.gsa_forward(q, k_, v, wg, L, top_k=k)
print('max err', np.abs(out.cpu().numpy() - ref['out']).max())
