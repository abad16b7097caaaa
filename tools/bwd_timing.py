"""Layer-backward timing on the B200: gsa_backward (attention part) and
gsa_project_backward (model_dim C) at the bench geometry for a list of view counts, CUDA
events on the launching stream, after a warm-up call. Prints one JSON line per size.
--ncu: one forward + one backward at the first size, for an ncu launch list."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_2603_08055_b200 as gsa  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--views", default="100,300,1000")
    ap.add_argument("--model-dim", type=int, default=1024)
    ap.add_argument("--iters", type=int, default=3)
    ap.add_argument("--ncu", action="store_true")
    a = ap.parse_args()
    for V in [int(x) for x in a.views.split(",")]:
        lt = bench.layout_for(V)
        L = gsa.build_token_layout(*lt)
        p = gsa.GsaParams(window_s=lt[4], top_k=bench.TOPK)
        q, k, v, wg = bench.synth_qkv(torch, V)
        out, ctx = gsa.gsa_forward(q, k, v, wg, L, p, context=True)
        plan = gsa.build_selection_plan(ctx.topk, L, p.variant, p.ref_stride)
        d_out = torch.randn_like(out)
        ws = gsa.Workspace()
        if a.ncu:
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStart()
            gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out, plan=plan, workspace=ws)
            torch.cuda.synchronize()
            torch.cuda.cudart().cudaProfilerStop()
            return
        gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out, plan=plan, workspace=ws)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            g = gsa.gsa_backward(q, k, v, wg, L, p, ctx, out, d_out, plan=plan, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        bwd_ms = e0.elapsed_time(e1) / a.iters
        # the same inputs through the forward for the ratio
        torch.cuda.synchronize()
        e0.record()
        for _ in range(a.iters):
            gsa.gsa_forward(q, k, v, wg, L, p, context=True, workspace=ws)
        e1.record()
        torch.cuda.synchronize()
        fwd_ms = e0.elapsed_time(e1) / a.iters
        H, M, d = q.shape
        C = a.model_dim
        x = torch.randn(M, C, device="cuda")
        w = [torch.randn(H, C, d, device="cuda") / C ** 0.5 for _ in range(3)]
        dq, dk, dv, _ = g
        gsa.project_backward(x, *w, dq, dk, dv)
        torch.cuda.synchronize()
        e0.record()
        gsa.project_backward(x, *w, dq, dk, dv)
        e1.record()
        torch.cuda.synchronize()
        proj_ms = e0.elapsed_time(e1)
        geo = bench.geometry(V)
        plan_entries = int(plan.window_ids.numel())
        # algorithmic FLOPs of the attention backward (FA2 accounting: 2 GEMMs to rebuild S and
        # dP, 3 for dQ/dK/dV; each 2*d per score): compressed W^2, special Ms*M, selection
        # entries * s^4 per head
        s4 = lt[4] ** 4
        flops = 5 * 2 * d * (H * geo["W"] ** 2 + H * geo["Ms"] * geo["M"] + plan_entries * s4)
        print(json.dumps(dict(views=V, tokens=M, windows=geo["W"], plan_entries=plan_entries, fwd_ms=round(fwd_ms, 3),
                              bwd_ms=round(bwd_ms, 3), proj_bwd_ms=round(proj_ms, 3), model_dim=C,
                              bwd_tflops=round(flops / bwd_ms / 1e9, 2),
                              proj_tflops=round(3 * 2 * 2 * M * C * H * d / proj_ms / 1e9, 2))), flush=True)
        del x, w, g, dq, dk, dv, q, k, v, out, ctx, plan, d_out, ws
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
