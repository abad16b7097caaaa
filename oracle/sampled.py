"""TEST INFRASTRUCTURE ONLY — sampled-row parity of a GPU layer forward at scale.

At the benchmarked sizes (V = 100 ... 1000 views, up to 1.3 M tokens) the full
reference layer is minutes to hours of CPU time, so parity is checked on a
seeded sample of (head, query-window) rows and special rows. For
every sampled row the UNMODIFIED reference (oracle/_ref, `gsa_ref_sampled_head`
in ref_harness.cpp) recomputes, from the same Q/K/V the GPU consumed:

* the guide scores against every key window with `scaled_dot` and the top-k with
  `naive_topk(_excluding)` (reference.hpp:236-247) -> compared BIT-EXACT, order
  included, with the GPU's indices;
* the compressed-branch row (softmax over all windows, reference.hpp:248-253);
* the plan row (build_selection_plan), the selection output of the window's
  s^2 queries (selection.hpp:100-133), gate and merge (layer.hpp:99-119,
  154-170) -> the final output rows, within the north-star tolerance;
* sampled special rows: dense attention over all M keys (layer.hpp:80-96).

Used by tests/test_scale_parity.py and by bench.py's cpu_baseline leg (after
the timed region). Never part of the measured path.
"""
from __future__ import annotations

import ctypes as C
import math
import os
import time

import numpy as np

from . import REF_SO, RefLib

_i32 = np.int32
_f32 = np.float32


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _lib():
    L = RefLib(REF_SO).lib
    L.gsa_ref_sampled_head.restype = C.c_int
    return L


def sample_rows(n: int, frac: float, seed: int, minimum: int = 1) -> np.ndarray:
    """Seeded sorted sample of ceil(frac * n) distinct row ids in [0, n)."""
    if n <= 0:
        return np.zeros(0, _i32)
    m = min(n, max(minimum, int(math.ceil(frac * n))))
    return np.sort(np.random.default_rng(seed).choice(n, m, replace=False)).astype(_i32)


def sampled_parity(q, k, v, w_g, lt, top_k, out, topk, *, variant=0, ref_stride=100, scale=0.0,
                   o_comp=None, lse_comp=None, o_sel=None, lse_sel=None, frac=0.01, spec_frac=0.0025,
                   seed=1234, heads=None, threads=None) -> dict:
    """Compare a GPU gsa_forward against the reference on sampled rows.

    q/k/v: device tensors [H][M][d] (bf16 or f32: the reference sees the same
    values upcast exactly); w_g device f32 [H][d][d]; out: the GPU's f32 output
    [H][M][d]; topk: the GPU's [H][W][k_eff]; o_comp/lse_comp/o_sel/lse_sel:
    optional context tensors. Returns the parity summary dict.
    """
    import torch

    ns, nf, gh, gw, s = lt
    H, M, d = q.shape
    s2 = s * s
    wpf = (gh // s) * (gw // s)
    W = nf * wpf
    heads = list(range(H)) if heads is None else list(heads)
    threads = threads or os.cpu_count() or 1
    L = _lib()
    t0 = time.perf_counter()
    # token ids (image rows) of every window, member order dr-outer dc-inner (layout.cpp:37-56)
    ww = gw // s
    rows_checked = spec_checked = topk_mismatch = 0
    first_bad = None
    num = den = 0.0
    max_abs = 0.0
    oc_num = oc_den = 0.0
    lse_c_max = 0.0
    sel_num = sel_den = 0.0
    lse_s_max = 0.0
    sp_num = sp_den = 0.0
    sp_max = 0.0
    k_eff = None
    for h in heads:
        wins = sample_rows(W, frac, seed + 7919 * h)
        specs = sample_rows(ns, spec_frac, seed + 104729 * h) if ns > 0 else np.zeros(0, _i32)
        qh, kh, vh = (np.ascontiguousarray(t[h].float().cpu().numpy()) for t in (q, k, v))
        wg = np.ascontiguousarray(w_g[h].float().cpu().numpy())
        n, ne = wins.size, specs.size
        ke_cap = max(1, min(top_k, W))
        r_topk = np.zeros((n, ke_cap), _i32)
        r_oc = np.zeros((n, d), _f32)
        r_lc = np.zeros(n, _f32)
        r_out = np.zeros((n, s2, d), _f32)
        r_sel = np.zeros((n, s2, d), _f32)
        r_lsel = np.zeros((n, s2), _f32)
        r_spec = np.zeros((max(ne, 1), d), _f32)
        ke = C.c_int()
        rc = L.gsa_ref_sampled_head(
            _p(qh), _p(kh), _p(vh), _p(wg), C.c_int(d), C.c_int(ns), C.c_int(nf), C.c_int(gh), C.c_int(gw),
            C.c_int(s), C.c_int(top_k), C.c_double(scale), C.c_int(variant), C.c_int(ref_stride), _p(wins),
            C.c_int(n), _p(specs), C.c_int(ne), C.c_int(threads), _p(r_topk), None, _p(r_oc), _p(r_lc),
            _p(r_out), _p(r_sel), _p(r_lsel), _p(r_spec), C.byref(ke))
        if rc != 0:
            raise RuntimeError(f"gsa_ref_sampled_head failed ({rc}): {L.gsa_ref_last_error().decode()}")
        k_eff = ke.value
        del qh, kh, vh
        # the GPU's rows for the same samples
        f, r = np.divmod(wins.astype(np.int64), wpf)
        wr, wc = np.divmod(r, ww)
        dr, dc = np.divmod(np.arange(s2), s)
        toks = (f[:, None] * gh * gw + (wr[:, None] * s + dr[None]) * gw + wc[:, None] * s + dc[None])  # [n][s2]
        dev = out.device
        wi = torch.from_numpy(wins.astype(np.int64)).to(dev)
        ti = torch.from_numpy((ns + toks.reshape(-1)).astype(np.int64)).to(dev)
        g_topk = topk[h].index_select(0, wi).cpu().numpy().astype(_i32)
        g_out = out[h].index_select(0, ti).float().cpu().numpy().reshape(n, s2, d)
        bad = np.nonzero((g_topk != r_topk[:, :k_eff]).any(1))[0]
        topk_mismatch += bad.size
        if bad.size and first_bad is None:
            first_bad = {"head": h, "window": int(wins[bad[0]]), "gpu": g_topk[bad[0]].tolist()[:8],
                         "ref": r_topk[bad[0], :k_eff].tolist()[:8]}
        rows_checked += n
        diff = (g_out - r_out).astype(np.float64)
        num += float((diff ** 2).sum())
        den += float((r_out.astype(np.float64) ** 2).sum())
        max_abs = max(max_abs, float(np.abs(diff).max()) if diff.size else 0.0)
        if o_comp is not None:
            g_oc = o_comp[h].index_select(0, wi).float().cpu().numpy()
            oc_num += float(((g_oc - r_oc).astype(np.float64) ** 2).sum())
            oc_den += float((r_oc.astype(np.float64) ** 2).sum())
        if lse_comp is not None:
            g_lc = lse_comp[h].index_select(0, wi).float().cpu().numpy()
            lse_c_max = max(lse_c_max, float(np.abs(g_lc - r_lc).max()))
        ti_img = torch.from_numpy(toks.reshape(-1).astype(np.int64)).to(dev)
        if o_sel is not None:
            g_sel = o_sel[h].index_select(0, ti_img).float().cpu().numpy().reshape(n, s2, d)
            sel_num += float(((g_sel - r_sel).astype(np.float64) ** 2).sum())
            sel_den += float((r_sel.astype(np.float64) ** 2).sum())
        if lse_sel is not None:
            g_ls = lse_sel[h].index_select(0, ti_img).float().cpu().numpy().reshape(n, s2)
            lse_s_max = max(lse_s_max, float(np.abs(g_ls - r_lsel).max()))
        if ne:
            si = torch.from_numpy(specs.astype(np.int64)).to(dev)
            g_sp = out[h].index_select(0, si).float().cpu().numpy()
            dsp = (g_sp - r_spec[:ne]).astype(np.float64)
            sp_num += float((dsp ** 2).sum())
            sp_den += float((r_spec[:ne].astype(np.float64) ** 2).sum())
            sp_max = max(sp_max, float(np.abs(dsp).max()))
            spec_checked += ne
    res = {
        "rows_checked": rows_checked, "rows_total": len(heads) * W, "frac": frac, "seed": seed, "k_eff": k_eff,
        "topk_mismatches": topk_mismatch, "max_abs": max_abs,
        "rel_l2": math.sqrt(num / den) if den > 0 else 0.0,
        "special_rows_checked": spec_checked,
        "special_max_abs": sp_max, "special_rel_l2": math.sqrt(sp_num / sp_den) if sp_den > 0 else 0.0,
        "checker": "oracle/_ref gsa_ref_sampled_head (unmodified reference: scaled_dot + naive_topk, "
                   "build_selection_plan, selection loop, gate/merge, special_token_attention)",
        "seconds": round(time.perf_counter() - t0, 1),
    }
    if o_comp is not None:
        res["o_comp_rel_l2"] = math.sqrt(oc_num / oc_den) if oc_den > 0 else 0.0
    if lse_comp is not None:
        res["lse_comp_max_abs"] = lse_c_max
    if o_sel is not None:
        res["o_sel_rel_l2"] = math.sqrt(sel_num / sel_den) if sel_den > 0 else 0.0
    if lse_sel is not None:
        res["lse_sel_max_abs"] = lse_s_max
    if first_bad is not None:
        res["first_mismatch"] = first_bad
    return res
