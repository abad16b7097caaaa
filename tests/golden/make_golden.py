"""Generate the committed golden fixtures from the UNMODIFIED reference.

Run here (where /root/reference exists and oracle/_ref/libgsa_ref.so is built):

    python tests/golden/make_golden.py

Small cases are stored whole (inputs as bf16 bit patterns, outputs as the
reference's float32 results). The parity-geometry cases (8 views, 16 heads)
are stored as SHA-256 digests of the top-k index arrays plus output checksums;
their inputs are regenerated from the seed by the oracle's counter RNG.
The reference path used is gsa_forward's body after project_qkv
(layer.hpp:194-229), i.e. oracle/_ref gsa_ref_forward.
"""
from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(HERE, "..", "..")))

from oracle import Layout, Oracle, RefLib, make_inputs  # noqa: E402

# name: (layout tuple, heads, top_k, variant, ref_stride, input kind)
SMALL = {
    "small_plain": ((3, 3, 8, 8, 4), 2, 2, 0, 100, "normal"),
    "small_hybrid": ((3, 3, 8, 8, 4), 2, 2, 1, 2, "normal"),
    "hybrid_frame0": ((5, 4, 8, 8, 4), 2, 3, 1, 100, "normal"),
    "sharp": ((5, 4, 12, 12, 4), 2, 5, 0, 100, "sharp"),
    "window2": ((1, 2, 8, 8, 2), 2, 3, 0, 100, "normal"),
    "dense_s1": ((0, 2, 8, 8, 1), 1, 128, 0, 100, "normal"),
    "ties": ((2, 2, 8, 8, 4), 2, 3, 0, 100, "ties"),
    "k_clamp": ((0, 1, 8, 12, 4), 2, 32, 0, 100, "normal"),
    "random_init": ((5, 2, 12, 12, 4), 2, 4, 0, 100, "random_init"),
    "clustered_init": ((5, 3, 8, 8, 4), 2, 3, 1, 100, "clustered_init"),
}

# parity geometry: 8 views, 5 specials/view, 36x36, s=4
PARITY = {
    "v8_normal": ((40, 8, 36, 36, 4), 16, 32, 0, 100, "normal"),
    "v8_sharp": ((40, 8, 36, 36, 4), 16, 32, 0, 100, "sharp"),
    "v8_hybrid": ((40, 8, 36, 36, 4), 16, 32, 1, 4, "normal"),
    "v8_uniform": ((40, 8, 36, 36, 4), 16, 32, 0, 100, "uniform"),
}


def bf16_bits(x: np.ndarray) -> np.ndarray:
    u = np.ascontiguousarray(x, np.float32).view(np.uint32)
    assert np.all((u & 0xFFFF) == 0), "inputs must be bf16-representable"
    return (u >> 16).astype(np.uint16)


def inputs_for(orc, ref, lt, heads, kind, seed=7):
    L = Layout(*lt)
    if kind in ("normal", "uniform"):
        return make_inputs(orc, L, heads=heads, dim=64, seed=seed, kind=kind)
    if kind == "sharp":
        return make_inputs(orc, L, heads=heads, dim=64, seed=seed, sharp=3.0)
    if kind == "ties":
        q, k, v, wg = make_inputs(orc, L, heads=heads, dim=64, seed=seed)
        k[0, :, :] = k[0, 0, :]  # head 0: every key identical -> every guide score ties
        return q, k, v, wg
    if kind in ("random_init", "clustered_init"):
        q, k, v, wg = ref.random_init(seed, lt, heads, 64, 128, clustered=(kind == "clustered_init"))
        return orc.bf16_round(q), orc.bf16_round(k), orc.bf16_round(v), wg
    raise ValueError(kind)


def digest(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def main() -> None:
    orc, ref = Oracle(), RefLib()
    for name, (lt, heads, k, variant, rs, kind) in SMALL.items():
        q, kk, v, wg = inputs_for(orc, ref, lt, heads, kind)
        r = ref.forward(q, kk, v, wg, lt, top_k=k, variant=variant, ref_stride=rs, threads=1)
        np.savez_compressed(
            os.path.join(HERE, f"{name}.npz"),
            layout=np.array(lt, np.int32), params=np.array([heads, k, variant, rs], np.int32),
            q=bf16_bits(q), k=bf16_bits(kk), v=bf16_bits(v), w_g=wg.astype(np.float32),
            out=r["out"], topk=r["topk"], qc=r["qc"], kc=r["kc"], vc=r["vc"], o_comp=r["o_comp"],
            lse_comp=r["lse_comp"], o_sel=r["o_sel"], lse_sel=r["lse_sel"], gate=r["gate"],
            lse_spec=r["lse_spec"])
        print(name, "k_eff", r["k_eff"])
    meta = {}
    for name, (lt, heads, k, variant, rs, kind) in PARITY.items():
        q, kk, v, wg = inputs_for(orc, ref, lt, heads, kind)
        r = ref.forward(q, kk, v, wg, lt, top_k=k, variant=variant, ref_stride=rs, threads=8)
        meta[name] = dict(layout=list(lt), heads=heads, top_k=k, variant=variant, ref_stride=rs,
                          kind=kind, seed=7, k_eff=r["k_eff"], topk_sha256=digest(r["topk"].astype(np.int32)),
                          qc_sha256=digest(r["qc"]), kc_sha256=digest(r["kc"]),
                          out_sum=float(r["out"].astype(np.float64).sum()),
                          out_abs_sum=float(np.abs(r["out"].astype(np.float64)).sum()),
                          stage_ms=r["stage_ms"])
        print(name, meta[name]["topk_sha256"][:16], {k_: round(v_, 1) for k_, v_ in r["stage_ms"].items()})
    with open(os.path.join(HERE, "parity_digests.json"), "w") as f:
        json.dump(meta, f, indent=1)


if __name__ == "__main__":
    main()
