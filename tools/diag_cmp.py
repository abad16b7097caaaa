import sys, numpy as np, torch
sys.path.insert(0,'/root/repo')
import paper_2603_08055_b200 as gsa
from oracle import Oracle
orc=Oracle()
W,k=int(sys.argv[1]),int(sys.argv[2])
rng=np.random.default_rng(W+k)
qc,kc,vc=(rng.standard_normal((3,W,64)).astype(np.float32) for _ in range(3))
o_ref,l_ref,i_ref,g_ref=orc.compress_topk(qc,kc,vc,k,0.125,guide=True)
r=gsa.fused_compressed_attention_topk(*(torch.from_numpy(x).cuda() for x in (qc,kc,vc)),k,0.125,keep_guide_scores=True)
torch.cuda.synchronize()
print('idx equal', np.array_equal(r.indices.cpu().numpy(), i_ref), 'out err', np.abs(r.out.cpu().numpy()-o_ref).max())
