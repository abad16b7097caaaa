import sys, numpy as np, torch
sys.path.insert(0,'/root/repo')
import paper_2603_08055_b200 as gsa
from oracle import Oracle
orc=Oracle()
for (mq,mk,grow) in [(77,4099,True),(77,4099,False),(128,1024,True),(128,2048,True)]:
    rng=np.random.default_rng(mq+mk)
    q=orc.bf16_round(rng.standard_normal((2,mq,64)).astype(np.float32))
    k=rng.standard_normal((2,mk,64)).astype(np.float32)
    if grow: k*=np.linspace(0.2,4.0,mk,dtype=np.float32)[None,:,None]
    k=orc.bf16_round(k); v=orc.bf16_round(rng.standard_normal((2,mk,64)).astype(np.float32))
    o_ref,l_ref=orc.dense_attention(q,k,v,0.125)
    dq,dk,dv=(torch.from_numpy(x).cuda().bfloat16() for x in (q,k,v))
    out,lse=gsa.tiled_attention(dq,dk,dv,0.125)
    o=out.float().cpu().numpy(); l=lse.cpu().numpy()
    err=np.abs(o-o_ref).max(-1)
    bad=np.argwhere(err>1e-3)
    print(mq,mk,grow,'max',err.max(),'nbad',len(bad),'rows',bad[:10].tolist(),'lse err',np.abs(l-l_ref).max())
    if len(bad):
        h,r=bad[0]; print(' out',o[h,r,:4],'ref',o_ref[h,r,:4],'lse',l[h,r],l_ref[h,r])
