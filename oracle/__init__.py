"""TEST INFRASTRUCTURE ONLY — Python bindings of the parity checkers.

* ``Oracle``  — the plain-C restatement of the reference GSA path
  (oracle/gsa_oracle.c, built into oracle/_build/libgsa_oracle.so).
* ``RefLib``  — the UNMODIFIED reference compiled from /root/reference into
  oracle/_ref/libgsa_ref.so (oracle/Makefile). The .so travels to the GPU box;
  the sources are only needed to build it.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline leg may
import this package. The product (paper_2603_08055_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libgsa_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libgsa_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")


def build() -> None:
    """Compile the C restatement (and oracle/_ref when /root/reference exists)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


class _Layout(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("num_special", "num_frames", "grid_h", "grid_w", "window_s")]


def _ptr_or_null(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


class Layout:
    """Mirror of layout.hpp:13-40 (pure integer arithmetic, used by tests)."""

    def __init__(self, num_special, num_frames, grid_h, grid_w, window_s):
        self.num_special, self.num_frames = num_special, num_frames
        self.grid_h, self.grid_w, self.window_s = grid_h, grid_w, window_s

    @property
    def tokens_per_frame(self):
        return self.grid_h * self.grid_w

    @property
    def image_tokens(self):
        return self.num_frames * self.tokens_per_frame

    @property
    def total_tokens(self):
        return self.num_special + self.image_tokens

    @property
    def windows_per_frame(self):
        return (self.grid_h // self.window_s) * (self.grid_w // self.window_s)

    @property
    def num_windows(self):
        return self.num_frames * self.windows_per_frame

    def tuple(self):
        return (self.num_special, self.num_frames, self.grid_h, self.grid_w, self.window_s)

    def c(self):
        return _Layout(*self.tuple())

    def tokens_of_window(self, w):
        s, gw = self.window_s, self.grid_w
        wpf, ww = self.windows_per_frame, gw // s
        f, r = divmod(w, wpf)
        wr, wc = divmod(r, ww)
        base = f * self.tokens_per_frame
        return [base + (wr * s + dr) * gw + wc * s + dc for dr in range(s) for dc in range(s)]

    def window_of_token(self, t):
        f, r = divmod(t, self.tokens_per_frame)
        row, col = divmod(r, self.grid_w)
        return f * self.windows_per_frame + (row // self.window_s) * (self.grid_w // self.window_s) + col // self.window_s


class Oracle:
    """ctypes binding of oracle/_build/libgsa_oracle.so."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_scaled_dot.restype = C.c_float
        L.orc_scaled_dot.argtypes = [_f32p, _f32p, C.c_int, C.c_float]
        L.orc_bf16_round.restype = C.c_float
        L.orc_bf16_round.argtypes = [C.c_float]
        L.orc_fill_normal.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_float, C.c_int, _f32p]
        L.orc_fill_uniform_bf16.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _f32p]
        L.orc_pool.argtypes = [_f32p, C.c_int, C.c_int, C.POINTER(_Layout), _f32p]
        L.orc_topk_row.argtypes = [_f32p, C.c_int, C.c_void_p, C.c_int, _i32p]
        L.orc_compress_topk.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                        C.c_float, C.c_void_p, C.c_void_p, C.c_int64, _f32p, _f32p,
                                        _i32p, C.c_void_p]
        L.orc_forced_windows.argtypes = [C.POINTER(_Layout), C.c_int, C.c_void_p, C.c_int]
        L.orc_build_plan.restype = C.c_int64
        L.orc_build_plan.argtypes = [_i32p, C.c_int, C.c_int, C.c_int, C.POINTER(_Layout), C.c_int,
                                     C.c_int, C.c_void_p, C.c_void_p]
        L.orc_block_sparse.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.POINTER(_Layout),
                                       _i64p, _i32p, C.c_float, C.c_void_p, C.c_int64, _f32p, _f32p]
        L.orc_dense_attention.argtypes = [_f32p, _f32p, _f32p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_float, _f32p, _f32p]
        L.orc_gate.argtypes = [_f32p, _f32p, C.c_int, C.c_int, C.c_int, _f32p]
        L.orc_gsa_forward.argtypes = [_f32p, _f32p, _f32p, _f32p, C.c_int, C.c_int, C.POINTER(_Layout),
                                      C.c_int, C.c_double, C.c_int, C.c_int, _f32p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p]

    # -- inputs ---------------------------------------------------------
    def normal(self, seed, tag, shape, mul=1.0, bf16=True):
        out = np.empty(int(np.prod(shape)), np.float32)
        self.lib.orc_fill_normal(seed, tag, out.size, mul, int(bf16), out)
        return out.reshape(shape)

    def uniform_bf16(self, seed, tag, shape):
        out = np.empty(int(np.prod(shape)), np.float32)
        self.lib.orc_fill_uniform_bf16(seed, tag, out.size, out)
        return out.reshape(shape)

    def bf16_round(self, x):
        x = f32(x)
        u = x.view(np.uint32).astype(np.uint64)
        u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
        return u.astype(np.uint32).view(np.float32).reshape(x.shape)

    # -- ops ------------------------------------------------------------
    def scaled_dot(self, a, b, scale=1.0):
        a, b = f32(a), f32(b)
        return self.lib.orc_scaled_dot(a, b, a.size, scale)

    def pool(self, x_img, layout: Layout):
        x_img = f32(x_img)
        H, _, d = x_img.shape
        out = np.empty((H, layout.num_windows, d), np.float32)
        self.lib.orc_pool(x_img, H, d, C.byref(layout.c()), out)
        return out

    def topk_row(self, scores, k, excluded=None):
        scores = f32(scores)
        out = np.empty(max(k, 1), np.int32)
        ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
        n = self.lib.orc_topk_row(scores, scores.size, _ptr_or_null(ex), k, out)
        if n < 0:
            raise FloatingPointError("NonFiniteInput")
        return out[:n]

    def compress_topk(self, qc, kc, vc, k, scale, excluded=None, rows=None, guide=False):
        qc, kc, vc = f32(qc), f32(kc), f32(vc)
        H, W, d = qc.shape
        ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
        sel = W - (0 if ex is None else int(ex.sum()))
        k_eff = min(k, sel)
        rr = None if rows is None else np.ascontiguousarray(rows, np.int64)
        n = H * W if rr is None else rr.size
        out = np.empty((n, d), np.float32)
        lse = np.empty(n, np.float32)
        idx = np.empty((n, max(k_eff, 1)), np.int32)
        g = np.empty((n, max(k_eff, 1)), np.float32) if guide else None
        rc = self.lib.orc_compress_topk(qc, kc, vc, H, W, d, k, scale, _ptr_or_null(ex),
                                        _ptr_or_null(rr), n, out, lse, idx, _ptr_or_null(g))
        if rc < 0:
            raise FloatingPointError("NonFiniteInput")
        idx = idx[:, :k_eff]
        if rr is None:
            out, lse, idx = out.reshape(H, W, d), lse.reshape(H, W), idx.reshape(H, W, k_eff)
        if guide:
            return out, lse, idx, g[:, :k_eff]
        return out, lse, idx

    def forced_windows(self, layout: Layout, ref_stride):
        n = self.lib.orc_forced_windows(C.byref(layout.c()), ref_stride, None, 0)
        if n < 0:
            raise ValueError("InvalidStride")
        out = np.empty(max(n, 1), np.int32)
        self.lib.orc_forced_windows(C.byref(layout.c()), ref_stride, out.ctypes.data_as(C.c_void_p), n)
        return out[:n]

    def build_plan(self, topk, layout: Layout, variant, ref_stride):
        topk = np.ascontiguousarray(topk, np.int32)
        H, W, k = topk.shape
        lc = layout.c()
        n = self.lib.orc_build_plan(topk, H, W, k, C.byref(lc), variant, ref_stride, None, None)
        if n < 0:
            raise ValueError("InvalidStride")
        offs = np.empty(H * W + 1, np.int64)
        ids = np.empty(max(n, 1), np.int32)
        self.lib.orc_build_plan(topk, H, W, k, C.byref(lc), variant, ref_stride,
                                offs.ctypes.data_as(C.c_void_p), ids.ctypes.data_as(C.c_void_p))
        return offs, ids[:n]

    def block_sparse(self, q_img, k_img, v_img, layout: Layout, offsets, ids, scale, rows=None):
        q_img, k_img, v_img = f32(q_img), f32(k_img), f32(v_img)
        H, Mi, d = q_img.shape
        s2 = layout.window_s ** 2
        offsets = np.ascontiguousarray(offsets, np.int64)
        ids = np.ascontiguousarray(ids, np.int32)
        if rows is None:
            out = np.empty((H, Mi, d), np.float32)
            lse = np.empty((H, Mi), np.float32)
            self.lib.orc_block_sparse(q_img, k_img, v_img, H, d, C.byref(layout.c()), offsets, ids,
                                      scale, None, 0, out, lse)
        else:
            rr = np.ascontiguousarray(rows, np.int64)
            out = np.empty((rr.size, s2, d), np.float32)
            lse = np.empty((rr.size, s2), np.float32)
            self.lib.orc_block_sparse(q_img, k_img, v_img, H, d, C.byref(layout.c()), offsets, ids,
                                      scale, rr.ctypes.data_as(C.c_void_p), rr.size, out, lse)
        return out, lse

    def dense_attention(self, q, k, v, scale):
        q, k, v = f32(q), f32(k), f32(v)
        H, mq, d = q.shape
        mk = k.shape[1]
        out = np.empty((H, mq, d), np.float32)
        lse = np.empty((H, mq), np.float32)
        self.lib.orc_dense_attention(q, k, v, H, mq, mk, d, scale, out, lse)
        return out, lse

    def gate(self, q_img, w_g):
        q_img, w_g = f32(q_img), f32(w_g)
        H, rows, d = q_img.shape
        g = np.empty_like(q_img)
        self.lib.orc_gate(q_img, w_g, H, rows, d, g)
        return g

    def gsa_forward(self, q, k, v, w_g, layout: Layout, top_k=32, scale=0.0, variant=0, ref_stride=100):
        q, k, v, w_g = f32(q), f32(k), f32(v), f32(w_g)
        H, M, d = q.shape
        W = layout.num_windows
        out = np.empty_like(q)
        topk = np.empty((H, W, max(1, top_k)), np.int32)
        o_comp = np.empty((H, W, d), np.float32)
        lse_comp = np.empty((H, W), np.float32)
        lse_sel = np.empty((H, layout.image_tokens), np.float32)
        k_eff = self.lib.orc_gsa_forward(q, k, v, w_g, H, d, C.byref(layout.c()), top_k, scale, variant,
                                         ref_stride, out, topk.ctypes.data_as(C.c_void_p),
                                         o_comp.ctypes.data_as(C.c_void_p),
                                         lse_comp.ctypes.data_as(C.c_void_p),
                                         lse_sel.ctypes.data_as(C.c_void_p))
        if k_eff < 0:
            raise RuntimeError(f"oracle gsa_forward failed: status {-k_eff}")
        topk = topk.reshape(-1)[: H * W * k_eff].reshape(H, W, k_eff)
        return dict(out=out, topk=topk, o_comp=o_comp, lse_comp=lse_comp, lse_sel=lse_sel, k_eff=k_eff)


class RefLib:
    """ctypes binding of the unmodified reference (oracle/_ref/libgsa_ref.so)."""

    ERRORS = {-1: "GsaError", -2: "ShapeMismatch", -3: "DivisibilityError", -4: "ZeroSizeError",
              -5: "IndexOutOfRange", -6: "NonFiniteInput", -7: "InvalidTiling", -8: "InvalidStride",
              -9: "EmptySelection", -99: "std::exception"}

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (needs /root/reference at build time)")
        L = self.lib = C.CDLL(path)
        L.gsa_ref_last_error.restype = C.c_char_p
        L.gsa_ref_scaled_dot.restype = C.c_float
        L.gsa_ref_scaled_dot.argtypes = [_f32p, _f32p, C.c_int, C.c_float]

    @staticmethod
    def available(path: str = REF_SO) -> bool:
        return os.path.exists(path)

    def _check(self, rc):
        if rc != 0:
            raise RuntimeError(f"{self.ERRORS.get(rc, rc)}: {self.lib.gsa_ref_last_error().decode()}")

    def status(self, rc):
        return self.ERRORS.get(rc, "ok" if rc == 0 else str(rc))

    @staticmethod
    def _p(a):
        return None if a is None else a.ctypes.data_as(C.c_void_p)

    def build_layout(self, *lt):
        w, t = C.c_int(), C.c_int()
        rc = self.lib.gsa_ref_build_layout(*[C.c_int(x) for x in lt], C.byref(w), C.byref(t))
        return rc, w.value, t.value

    def window_of_token(self, lt, t):
        o = C.c_int()
        self._check(self.lib.gsa_ref_window_of_token(*[C.c_int(x) for x in lt], C.c_int(t), C.byref(o)))
        return o.value

    def tokens_of_window(self, lt, w):
        o = np.empty(lt[4] ** 2, np.int32)
        self._check(self.lib.gsa_ref_tokens_of_window(*[C.c_int(x) for x in lt], C.c_int(w), self._p(o)))
        return o

    def scaled_dot(self, a, b, scale=1.0):
        a, b = f32(a), f32(b)
        return self.lib.gsa_ref_scaled_dot(a, b, a.size, C.c_float(scale))

    def naive_topk(self, scores, k, excluded=None):
        scores = f32(scores)
        out = np.empty(max(1, scores.size), np.int32)
        cnt = C.c_int()
        ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
        self._check(self.lib.gsa_ref_naive_topk(self._p(scores), C.c_int(scores.size), self._p(ex),
                                                C.c_int(k), self._p(out), C.byref(cnt)))
        return out[: cnt.value]

    def pool(self, x_img, lt):
        x_img = f32(x_img)
        H, _, d = x_img.shape
        W = self.build_layout(*lt)[1]
        out = np.empty((H, W, d), np.float32)
        self._check(self.lib.gsa_ref_pool(self._p(x_img), C.c_int(H), C.c_int(d), *[C.c_int(x) for x in lt], self._p(out)))
        return out

    def upsample(self, coarse, lt):
        coarse = f32(coarse)
        H, W, d = coarse.shape
        Mi = self.build_layout(*lt)[2]
        out = np.empty((H, Mi, d), np.float32)
        self._check(self.lib.gsa_ref_upsample(self._p(coarse), C.c_int(H), C.c_int(d), *[C.c_int(x) for x in lt], self._p(out)))
        return out

    def compress(self, qc, kc, vc, k, scale, bm=16, bn=16, excluded=None, threads=8, guide=False):
        qc, kc, vc = f32(qc), f32(kc), f32(vc)
        H, W, d = qc.shape
        ex = None if excluded is None else np.ascontiguousarray(excluded, np.uint8)
        out = np.empty((H, W, d), np.float32)
        lse = np.empty((H, W), np.float32)
        idx = np.empty(H * W * max(1, min(k, W)), np.int32)
        g = np.empty(H * W * max(1, min(k, W)), np.float64) if guide else None
        ke = C.c_int()
        self._check(self.lib.gsa_ref_compress(self._p(qc), self._p(kc), self._p(vc), C.c_int(H), C.c_int(W),
                                              C.c_int(d), C.c_int(k), C.c_float(scale), C.c_int(bm), C.c_int(bn),
                                              self._p(ex), C.c_int(threads), self._p(out), self._p(lse),
                                              self._p(idx), self._p(g), C.byref(ke)))
        k_eff = ke.value
        idx = idx[: H * W * k_eff].reshape(H, W, k_eff)
        if guide:
            return out, lse, idx, g[: H * W * k_eff].reshape(H, W, k_eff)
        return out, lse, idx

    def plan(self, topk, lt, variant, ref_stride):
        topk = np.ascontiguousarray(topk, np.int32)
        H, W, k = topk.shape
        n = C.c_int64()
        args = [self._p(topk), C.c_int(H), C.c_int(W), C.c_int(k), *[C.c_int(x) for x in lt],
                C.c_int(variant), C.c_int(ref_stride)]
        self._check(self.lib.gsa_ref_plan(*args, None, None, C.byref(n)))
        offs = np.empty(H * W + 1, np.int64)
        ids = np.empty(max(1, n.value), np.int32)
        self._check(self.lib.gsa_ref_plan(*args, self._p(offs), self._p(ids), C.byref(n)))
        return offs, ids[: n.value]

    def forced_windows(self, lt, ref_stride):
        cnt = C.c_int()
        self._check(self.lib.gsa_ref_forced_windows(*[C.c_int(x) for x in lt], C.c_int(ref_stride), None, C.byref(cnt)))
        out = np.empty(max(1, cnt.value), np.int32)
        self._check(self.lib.gsa_ref_forced_windows(*[C.c_int(x) for x in lt], C.c_int(ref_stride), self._p(out), C.byref(cnt)))
        return out[: cnt.value]

    def block_sparse(self, q_img, k_img, v_img, lt, offsets, ids, scale, threads=8):
        q_img, k_img, v_img = f32(q_img), f32(k_img), f32(v_img)
        H, Mi, d = q_img.shape
        offsets = np.ascontiguousarray(offsets, np.int64)
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.empty((H, Mi, d), np.float32)
        lse = np.empty((H, Mi), np.float32)
        self._check(self.lib.gsa_ref_block_sparse(self._p(q_img), self._p(k_img), self._p(v_img), C.c_int(H),
                                                  C.c_int(d), *[C.c_int(x) for x in lt], self._p(offsets),
                                                  self._p(ids), C.c_float(scale), C.c_int(threads),
                                                  self._p(out), self._p(lse)))
        return out, lse

    def masked_attention(self, q_img, k_img, v_img, lt, offsets, ids, scale):
        """masked_image_attention (reference.hpp:120-170) -> (out, denominators f64)."""
        q_img, k_img, v_img = f32(q_img), f32(k_img), f32(v_img)
        H, Mi, d = q_img.shape
        offsets = np.ascontiguousarray(offsets, np.int64)
        ids = np.ascontiguousarray(ids, np.int32)
        out = np.empty((H, Mi, d), np.float32)
        den = np.empty((H, Mi), np.float64)
        self._check(self.lib.gsa_ref_masked_attention(self._p(q_img), self._p(k_img), self._p(v_img), C.c_int(H),
                                                      C.c_int(d), *[C.c_int(x) for x in lt], self._p(offsets),
                                                      self._p(ids), C.c_float(scale), self._p(out), self._p(den)))
        return out, den

    def tiled_attention(self, q, k, v, scale, bm=16, bn=16, threads=8):
        q, k, v = f32(q), f32(k), f32(v)
        H, mq, d = q.shape
        mk = k.shape[1]
        out = np.empty((H, mq, d), np.float32)
        lse = np.empty((H, mq), np.float32)
        self._check(self.lib.gsa_ref_tiled_attention(self._p(q), self._p(k), self._p(v), C.c_int(H), C.c_int(mq),
                                                     C.c_int(mk), C.c_int(d), C.c_float(scale), C.c_int(bm),
                                                     C.c_int(bn), C.c_int(threads), self._p(out), self._p(lse)))
        return out, lse

    def full_attention(self, q, k, v, scale):
        q, k, v = f32(q), f32(k), f32(v)
        H, mq, d = q.shape
        out = np.empty((H, mq, d), np.float32)
        self._check(self.lib.gsa_ref_full_attention(self._p(q), self._p(k), self._p(v), C.c_int(H), C.c_int(mq),
                                                    C.c_int(k.shape[1]), C.c_int(d), C.c_float(scale), self._p(out)))
        return out

    def gate(self, q_img, w_g):
        q_img, w_g = f32(q_img), f32(w_g)
        H, rows, d = q_img.shape
        g = np.empty_like(q_img)
        self._check(self.lib.gsa_ref_gate(self._p(q_img), self._p(w_g), C.c_int(H), C.c_int(rows), C.c_int(d), self._p(g)))
        return g

    def forward(self, q, k, v, w_g, lt, top_k=32, scale=0.0, variant=0, ref_stride=100, bm=16, bn=16,
                threads=8, context=True):
        """The reference fused CPU layer from projected Q/K/V (layer.hpp:194-229)."""
        q, k, v, w_g = f32(q), f32(k), f32(v), f32(w_g)
        H, M, d = q.shape
        _, W, Mi = self.build_layout(*lt)
        out = np.empty_like(q)
        ctx = {}
        if context:
            ctx = dict(qc=np.empty((H, W, d), np.float32), kc=np.empty((H, W, d), np.float32),
                       vc=np.empty((H, W, d), np.float32), o_comp=np.empty((H, W, d), np.float32),
                       lse_comp=np.empty((H, W), np.float32),
                       topk=np.empty(H * W * max(1, top_k), np.int32),
                       o_sel=np.empty((H, Mi, d), np.float32), lse_sel=np.empty((H, Mi), np.float32),
                       gate=np.empty((H, Mi, d), np.float32), lse_spec=np.empty((H, lt[0]), np.float32))
        ke = C.c_int()
        ms = np.zeros(7, np.float64)
        g = lambda n: self._p(ctx.get(n))  # noqa: E731
        self._check(self.lib.gsa_ref_forward(
            self._p(q), self._p(k), self._p(v), self._p(w_g), C.c_int(H), C.c_int(d), *[C.c_int(x) for x in lt],
            C.c_int(top_k), C.c_double(scale), C.c_int(variant), C.c_int(ref_stride), C.c_int(bm), C.c_int(bn),
            C.c_int(threads), self._p(out), g("qc"), g("kc"), g("vc"), g("o_comp"), g("lse_comp"), g("topk"),
            C.byref(ke), g("o_sel"), g("lse_sel"), g("gate"), g("lse_spec"), self._p(ms)))
        ctx["k_eff"] = ke.value
        if context:
            ctx["topk"] = ctx["topk"][: H * W * ke.value].reshape(H, W, ke.value)
        ctx["stage_ms"] = dict(zip(["partition", "special", "pool", "compress", "plan", "select", "gate_merge"], ms))
        ctx["out"] = out
        return ctx

    def reference_gsa(self, q, k, v, w_g, lt, top_k=32, scale=0.0, variant=0, ref_stride=100):
        q, k, v, w_g = f32(q), f32(k), f32(v), f32(w_g)
        H, M, d = q.shape
        out = np.empty_like(q)
        self._check(self.lib.gsa_ref_reference_gsa(self._p(q), self._p(k), self._p(v), self._p(w_g), C.c_int(H),
                                                   C.c_int(d), *[C.c_int(x) for x in lt], C.c_int(top_k),
                                                   C.c_double(scale), C.c_int(variant), C.c_int(ref_stride),
                                                   self._p(out)))
        return out

    def project(self, x, w_q, w_k, w_v):
        """project_qkv (layer.hpp:48-76): x [tokens][C], w_* [H][C][d] -> q, k, v [H][tokens][d]."""
        x, w_q, w_k, w_v = (np.ascontiguousarray(a, np.float32) for a in (x, w_q, w_k, w_v))
        tokens, C_ = x.shape
        H, _, d = w_q.shape
        q, k, v = (np.empty((H, tokens, d), np.float32) for _ in range(3))
        self._check(self.lib.gsa_ref_project(self._p(x), C.c_int(tokens), C.c_int(C_), self._p(w_q), self._p(w_k),
                                             self._p(w_v), C.c_int(H), C.c_int(d), self._p(q), self._p(k), self._p(v)))
        return q, k, v

    def backward(self, x, w_q, w_k, w_v, w_g, lt, d_out, top_k=32, scale=0.0, variant=0, ref_stride=100,
                 threads=8, f64=False):
        """gsa_forward (layer.hpp:177-230) + gsa_backward (gradients.hpp:54-265) from X and the
        weights: the forward output, its saved context (q/k/v, qc/kc/vc, o_comp, lse_comp, topk,
        o_sel, lse_sel, gate, lse_spec) and the gradients dx, dw_q, dw_k, dw_v, dw_g."""
        x, w_q, w_k, w_v, w_g, d_out = (np.ascontiguousarray(a, np.float32) for a in (x, w_q, w_k, w_v, w_g, d_out))
        M, Cm = x.shape
        H, _, d = w_q.shape
        _, W, Mi = self.build_layout(*lt)
        e = lambda *s: np.empty(s, np.float32)  # noqa: E731
        r = dict(out=e(H, M, d), q=e(H, M, d), k=e(H, M, d), v=e(H, M, d), qc=e(H, W, d), kc=e(H, W, d),
                 vc=e(H, W, d), o_comp=e(H, W, d), lse_comp=e(H, W), topk=np.empty(H * W * max(1, top_k), np.int32),
                 o_sel=e(H, Mi, d), lse_sel=e(H, Mi), gate=e(H, Mi, d), lse_spec=e(H, lt[0]), dx=e(M, Cm),
                 dw_q=e(H, Cm, d), dw_k=e(H, Cm, d), dw_v=e(H, Cm, d), dw_g=e(H, d, d))
        ke = C.c_int()
        ms = np.zeros(2, np.float64)
        p = lambda n: self._p(r[n])  # noqa: E731
        self._check(self.lib.gsa_ref_backward(
            self._p(x), C.c_int(Cm), self._p(w_q), self._p(w_k), self._p(w_v), self._p(w_g), C.c_int(H), C.c_int(d),
            *[C.c_int(a) for a in lt], C.c_int(top_k), C.c_double(scale), C.c_int(variant), C.c_int(ref_stride),
            C.c_int(threads), C.c_int(int(f64)), self._p(d_out), p("out"), p("q"), p("k"), p("v"), p("qc"), p("kc"),
            p("vc"), p("o_comp"), p("lse_comp"), p("topk"), C.byref(ke), p("o_sel"), p("lse_sel"), p("gate"),
            p("lse_spec"), p("dx"), p("dw_q"), p("dw_k"), p("dw_v"), p("dw_g"), self._p(ms)))
        r["k_eff"] = ke.value
        r["topk"] = r["topk"][: H * W * ke.value].reshape(H, W, ke.value)
        r["ms"] = dict(forward=ms[0], backward=ms[1])
        return r

    def random_init(self, seed, lt, heads, dim, model_dim, clustered=False):
        M = self.build_layout(*lt)[2] + lt[0]
        q, k, v = (np.empty((heads, M, dim), np.float32) for _ in range(3))
        w_g = np.empty((heads, dim, dim), np.float32)
        self._check(self.lib.gsa_ref_random_init(C.c_uint64(seed), *[C.c_int(x) for x in lt], C.c_int(heads),
                                                 C.c_int(dim), C.c_int(model_dim), C.c_int(int(clustered)),
                                                 self._p(q), self._p(k), self._p(v), self._p(w_g)))
        return q, k, v, w_g


def make_inputs(orc: Oracle, layout: Layout, heads=16, dim=64, seed=7, kind="normal", sharp=1.0):
    """Synthetic post-projection inputs of SURVEY §8(d): Q/K/V on streams 11/12/13,
    bf16-representable; W_g = N(0,1)/8 on stream 5 (workload.hpp:104 scaling)."""
    M = layout.total_tokens
    shape = (heads, M, dim)
    if kind == "normal":
        q = orc.normal(seed, 11, shape, 1.0, True)
        k = orc.normal(seed, 12, shape, 1.0, True)
        v = orc.normal(seed, 13, shape, 1.0, True)
    elif kind == "uniform":
        q = orc.uniform_bf16(seed, 11, shape)
        k = orc.uniform_bf16(seed, 12, shape)
        v = orc.uniform_bf16(seed, 13, shape)
    else:
        raise ValueError(kind)
    if sharp != 1.0:
        q = orc.bf16_round(q * np.float32(sharp))
        k = orc.bf16_round(k * np.float32(sharp))
    w_g = orc.normal(seed, 5, (heads, dim, dim), 1.0 / np.sqrt(dim), False)
    return q, k, v, w_g
