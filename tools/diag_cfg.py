"""Repro of one random SPEC config (tests/test_spec_properties.py) with launch-blocking errors."""
import os, sys
os.environ.setdefault("CUDA_LAUNCH_BLOCKING", "1")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import torch
import paper_2603_08055_b200 as gsa
from test_spec_properties import random_config, bf16r, dev
block = int(sys.argv[1]) if len(sys.argv) > 1 else 2
rng = np.random.default_rng(574 + 1000 * block)
for i in range(25):
    lt, k, variant, ref_stride, H, d = random_config(rng)
    M = lt[0] + lt[1] * lt[2] * lt[3]
    dt = torch.float32 if rng.random() < 0.5 else torch.bfloat16
    q, kk, v = (rng.standard_normal((H, M, d)).astype(np.float32) for _ in range(3))
    if dt == torch.bfloat16:
        q, kk, v = bf16r(q), bf16r(kk), bf16r(v)
    wg = (rng.standard_normal((H, d, d)) / np.sqrt(d)).astype(np.float32)
    L = gsa.build_token_layout(*lt)
    p = gsa.GsaParams(window_s=lt[4], top_k=k, variant=variant, ref_stride=ref_stride)
    try:
        out, ctx = gsa.gsa_forward(dev(q, dt), dev(kk, dt), dev(v, dt), dev(wg, torch.float32), L, p, context=True)
        torch.cuda.synchronize()
        print(i, "ok", lt, k, variant, ref_stride, H, d, dt)
    except Exception as e:
        print(i, "FAIL", lt, k, variant, ref_stride, H, d, dt, e)
        break
