"""Shared fixtures. `-m gpu` tests need a B200 and libgsa_sm100.so; everything
else runs on the CPU box (oracle, reference harness, host-side ABI checks)."""
from __future__ import annotations

import glob
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")

# Attention outputs of the tensor-core kernels: P (and V, scaled per head by a power of
# two) enter the P.V products as fp16, so each output carries |dO| <= 2^-12 * max|v| of P
# rounding (observed ~1e-4 .. 2e-4 abs on N(0,1) values). Asserted well inside the north
# star's max-abs 2e-2 / rel-L2 1e-3 (BASELINE.json): max-abs 1e-3, rel-L2 1e-3.
P16_ABS, P16_REL = 1e-3, 1e-3


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA B200 (sm_100a) device")


@pytest.fixture(scope="session")
def orc():
    from oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    from oracle import RefLib
    if not RefLib.available():
        pytest.skip("oracle/_ref/libgsa_ref.so not built (needs /root/reference at build time)")
    return RefLib()


def bf16_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << 16).view(np.float32)


def load_golden(name: str) -> dict:
    z = np.load(os.path.join(GOLDEN, f"{name}.npz"))
    d = {k: z[k] for k in z.files}
    for key in ("q", "k", "v"):
        d[key] = bf16_to_f32(d[key])
    d["layout"] = tuple(int(x) for x in d["layout"])
    heads, top_k, variant, ref_stride = (int(x) for x in d["params"])
    d.update(heads=heads, top_k=top_k, variant=variant, ref_stride=ref_stride)
    return d


GOLDEN_NAMES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(GOLDEN, "*.npz")))


def rel_l2(a, b) -> float:
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))
