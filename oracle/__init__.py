"""CPU oracle for the GELU-less INT8 Swin MLP sub-layer (arXiv 2402.01169).

TEST INFRASTRUCTURE.  Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package.  It shares no
code with the CUDA product path (paper_2402_01169_b200) and the product path
never imports it.

The arithmetic lives in oracle_mlp.c (plain C loops, one rounding per written
fp32 op, LayerNorm statistics in double); this module only marshals numpy
arrays through ctypes.  Step names O0..O7 follow SURVEY.md §8(c) and cite
PAPER.md Fig. 1 (lines 72-86) and the GELU-less section (lines 244-247, 326-328).

Parity status per function: every step is pinned by
tests/test_oracle_pins.py (brute force, closed forms, invariants, library
cross-checks, exhaustive grid round trips).  The composed layer (O7) has no
worked example in the paper ("parity unpinned" by the paper itself); it is
pinned only through its pinned steps and a float-reference sanity budget.
"""
import ctypes
import os

import numpy as np

from . import build as _build

ACT_RELU = 0
ACT_GELU = 1
ACT_SHIFT_GELU = 2

_lib = None


def lib():
    global _lib
    if _lib is None:
        path = _build.build()
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        i32, i64, f32 = ctypes.c_int32, ctypes.c_int64, ctypes.c_float
        L.oracle_fold_constants.argtypes = [i32, i32, f32, P, f32, P, f32, P, P, P, P]
        L.oracle_fold_constants.restype = None
        L.oracle_gemm_i8.argtypes = [P, i64, P, i64, i32, P, i32, i32, P, i32]
        L.oracle_gemm_i8.restype = i32
        L.oracle_ep5.argtypes = [P, i64, i32, P, P, f32, i32, i32, P, P]
        L.oracle_ep5.restype = None
        L.oracle_ep6.argtypes = [P, i64, i32, P, P, P, P, f32, i32, P, P, f32, f32, i32, P, P, P]
        L.oracle_ep6.restype = None
        L.oracle_ep5_shiftgelu.argtypes = [P, i64, i32, P, P, f32, f32, i32, P, P]
        L.oracle_ep5_shiftgelu.restype = None
        L.oracle_mlp.argtypes = [P, P, P, P, i64, i32, P, P, P, P, P, P]
        L.oracle_mlp.restype = i32
        L.oracle_max_threads.restype = i32
        L.oracle_q.argtypes = [P, i64, f32, i32, P]
        L.oracle_q.restype = None
        L.oracle_dq.argtypes = [P, i64, f32, i32, P]
        L.oracle_dq.restype = None
        # attention half (oracle_attn.c)
        L.oracle_window_src_row.argtypes = [i64, i32, i32, i32, i32]
        L.oracle_window_src_row.restype = i64
        L.oracle_op1.argtypes = [P, i32, i32, i32, i32, i32, i32, P, P, f32, f32, i32, P, i64, P, P]
        L.oracle_op1.restype = None
        L.oracle_qkv.argtypes = [P, i64, i32, i32, P, P, P, f32, f32, f32, f32, P, P]
        L.oracle_qkv.restype = None
        L.oracle_rel_bias.argtypes = [P, i32, i32, P]
        L.oracle_rel_bias.restype = None
        L.oracle_shift_mask.argtypes = [i32, i32, i32, i32, P]
        L.oracle_shift_mask.restype = None
        L.oracle_attn_fold.argtypes = [f32, f32, f32, f32, i32, P, P, P]
        L.oracle_attn_fold.restype = None
        L.oracle_attn.argtypes = [P, i64, i32, i32, i32, i32, i32, i32, f32, P, P, f32, f32, i32, P, i64, P, P]
        L.oracle_attn.restype = None
        _lib = L
    return _lib


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _c(a, dt):
    return None if a is None else np.ascontiguousarray(a, dtype=dt)


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def quantize(x, s, z):
    """Q: clamp(rne(fl(x * fl(1/s))) + z, -128, 127)."""
    x = _c(np.atleast_1d(x), np.float32)
    q = np.empty(x.shape, np.int8)
    inv = np.float32(1.0) / np.float32(s)
    lib().oracle_q(_p(x), x.size, float(inv), int(z), _p(q))
    return q


def dequantize(q, s, z):
    """dQ: fl(fl(q - z) * s)."""
    q = _c(np.atleast_1d(q), np.int8)
    x = np.empty(q.shape, np.float32)
    lib().oracle_dq(_p(q), q.size, float(s), int(z), _p(x))
    return x


def fold_constants(s_x, s_w1, s_h, s_w2, s_y):
    """O0: m1 = fl(s_x*s_w1), inv_h = fl(1/s_h), m2 = fl(s_h*s_w2), inv_y = fl(1/s_y)."""
    s_w1 = _c(s_w1, np.float32); s_w2 = _c(s_w2, np.float32)
    H, C = s_w1.shape[0], s_w2.shape[0]
    m1 = np.empty(H, np.float32); m2 = np.empty(C, np.float32)
    ih = np.empty(1, np.float32); iy = np.empty(1, np.float32)
    lib().oracle_fold_constants(C, H, float(s_x), _p(s_w1), float(s_h), _p(s_w2), float(s_y),
                                _p(m1), _p(ih), _p(m2), _p(iy))
    return m1, float(ih[0]), m2, float(iy[0])


def gemm_i8(X, W, zp, rows=None, nthreads=0):
    """O1/O3: A[t,n] = sum_k (X[t,k]-zp)*W[n,k], int64-accumulated, checked to fit int32."""
    X = _c(X, np.int8); W = _c(W, np.int8)
    K = X.shape[1]
    assert W.shape[1] == K
    N = W.shape[0]
    r = None if rows is None else _c(rows, np.int64)
    nrows = X.shape[0] if r is None else r.shape[0]
    A = np.empty((nrows, N), np.int32)
    st = lib().oracle_gemm_i8(_p(X), K, _p(r), nrows, K, _p(W), N, int(zp), _p(A), int(nthreads))
    if st != 0:
        raise OverflowError("int32 accumulator overflow in oracle_gemm_i8")
    return A


def ep5(A1, m1, b1, inv_h, z_h, act=ACT_RELU, return_pre=False):
    """O2/O2': Hq = clamp(rne(fl(act(fmaf(fl(A1), m1, b1)) * inv_h)) + z_h)."""
    A1 = _c(A1, np.int32); m1 = _c(m1, np.float32); b1 = _c(b1, np.float32)
    T, H = A1.shape
    Hq = np.empty((T, H), np.int8)
    pre = np.empty((T, H), np.float32) if return_pre else None
    lib().oracle_ep5(_p(A1), T, H, _p(m1), _p(b1), float(inv_h), int(z_h), int(act), _p(Hq), _p(pre))
    return (Hq, pre) if return_pre else Hq


def ep5_shiftgelu(A1, m1, b1, s_g, inv_h, z_h, return_I=False):
    """O2'': the I-ViT shift-GELU control (R28): Hq from A1 with the per-row max."""
    A1 = _c(A1, np.int32); m1 = _c(m1, np.float32); b1 = _c(b1, np.float32)
    T, H = A1.shape
    Hq = np.empty((T, H), np.int8)
    I = np.empty((T, H), np.int32) if return_I else None
    lib().oracle_ep5_shiftgelu(_p(A1), T, H, _p(m1), _p(b1), float(s_g), float(inv_h), int(z_h), _p(Hq), _p(I))
    return (Hq, I) if return_I else Hq


def ep6(A2, m2, b2, X, s_x, z_x, gamma, beta, eps, inv_y, z_y, R=None):
    """O4-O6: returns (Y int8, yhat fp32, z fp32)."""
    A2 = _c(A2, np.int32); m2 = _c(m2, np.float32); b2 = _c(b2, np.float32)
    X = _c(X, np.int8); R = _c(R, np.float32)
    gamma = _c(gamma, np.float32); beta = _c(beta, np.float32)
    T, C = A2.shape
    Y = np.empty((T, C), np.int8); yh = np.empty((T, C), np.float32); z = np.empty((T, C), np.float32)
    lib().oracle_ep6(_p(A2), T, C, _p(m2), _p(b2), _p(R), _p(X), float(s_x), int(z_x),
                     _p(gamma), _p(beta), float(eps), float(inv_y), int(z_y), _p(z), _p(yh), _p(Y))
    return Y, yh, z


def proj_op4(P, A_in, R):
    """SURVEY.md §8(f) NEXT-2, Fig. 1 lines 63-70 (Proj GEMM -> fused op #4: dQ -> Proj
    Bias -> Add (Residual) -> Q), with LN2 before the Q (reading R18: the Swin block is
    pre-norm, so FC1's input is LN2(x + proj)).  Composition of the pinned steps, in this order:
      O3  A[t,c] = sum_k (A_in[t,k] - z_a) * W[c,k]             (gemm_i8)
      O0  m[c] = fl(s_a * s_w[c]), inv_y = fl(1/s_y)              (fold_constants, h-slot = s_a)
      O4-O6 with the fp32 shortcut R: z = fl(fmaf(fl(A), m, b) + R); yhat = LN2(z); Y = Q_y(yhat)
    Returns (Y int8, yhat fp32, z fp32, A int32)."""
    A = gemm_i8(A_in, P.w, P.z_a)
    C = P.C
    _, _, m, inv_y = fold_constants(1.0, np.ones(C, np.float32), P.s_a, P.s_w, P.s_y)
    Y, yhat, z = ep6(A, m, P.b, np.zeros_like(A_in), 1.0, 0, P.gamma, P.beta, P.eps, inv_y, P.z_y, R=R)
    return Y, yhat, z, A


class _Layer(ctypes.Structure):
    _fields_ = [("C", ctypes.c_int32), ("H", ctypes.c_int32), ("act", ctypes.c_int32),
                ("s_x", ctypes.c_float), ("z_x", ctypes.c_int32),
                ("w1", ctypes.c_void_p), ("s_w1", ctypes.c_void_p), ("b1", ctypes.c_void_p),
                ("s_h", ctypes.c_float), ("z_h", ctypes.c_int32),
                ("w2", ctypes.c_void_p), ("s_w2", ctypes.c_void_p), ("b2", ctypes.c_void_p),
                ("gamma", ctypes.c_void_p), ("beta", ctypes.c_void_p), ("eps", ctypes.c_float),
                ("s_y", ctypes.c_float), ("z_y", ctypes.c_int32), ("s_g", ctypes.c_float)]


def mlp(layer, X, R=None, rows=None, nthreads=0, taps=False):
    """O7: whole layer on the selected rows.  `layer` is a synth.Layer (or any
    object with the same attributes).  Returns Y [nrows, C] int8, or a dict of
    all taps (acc1, hidden, acc2, yhat, z, y) when taps=True."""
    C, H = layer.C, layer.H
    keep = []

    def arr(a, dt):
        if a is None:
            return None
        a = np.ascontiguousarray(a, dtype=dt)
        keep.append(a)
        return a

    w1 = arr(layer.w1, np.int8); s_w1 = arr(layer.s_w1, np.float32); b1 = arr(layer.b1, np.float32)
    w2 = arr(layer.w2, np.int8); s_w2 = arr(layer.s_w2, np.float32); b2 = arr(layer.b2, np.float32)
    g = arr(layer.gamma, np.float32); bt = arr(layer.beta, np.float32)
    L = _Layer(C, H, int(layer.act), float(layer.s_x), int(layer.z_x), _p(w1), _p(s_w1), _p(b1),
               float(layer.s_h), int(layer.z_h), _p(w2), _p(s_w2), _p(b2), _p(g), _p(bt),
               float(layer.eps), float(layer.s_y), int(layer.z_y), float(getattr(layer, "s_g", 0.0) or 0.0))
    X = arr(X, np.int8); R = arr(R, np.float32)
    assert X.shape[1] == C
    r = None if rows is None else arr(rows, np.int64)
    n = X.shape[0] if r is None else r.shape[0]
    Y = np.empty((n, C), np.int8)
    if taps:
        a1 = np.empty((n, H), np.int32); h = np.empty((n, H), np.int8)
        a2 = np.empty((n, C), np.int32); yh = np.empty((n, C), np.float32); z = np.empty((n, C), np.float32)
    else:
        a1 = h = a2 = yh = z = None
    st = lib().oracle_mlp(ctypes.byref(L), _p(X), _p(R), _p(r), n, int(nthreads), _p(Y),
                          _p(a1), _p(h), _p(a2), _p(yh), _p(z))
    if st != 0:
        raise OverflowError("int32 accumulator overflow in oracle_mlp")
    if taps:
        return {"acc1": a1, "hidden": h, "acc2": a2, "yhat": yh, "z": z, "y": Y}
    return Y


# ---- attention half of the block (oracle_attn.c) -------------

def window_src_row(r, Hs, Ws, M, s):
    """Raster row (b*Hs*Ws + y*Ws + x) of window-ordered row r (readings R21, R22)."""
    return int(lib().oracle_window_src_row(int(r), int(Hs), int(Ws), int(M), int(s)))


def op1(x, gamma, beta, eps, s_q, z_q, M, shift, rows=None, return_yhat=False):
    """Fused op #1: LayerNorm -> window shift -> Q.  x: fp32 [B][Hs][Ws][C].
    Returns int8 [nrows][C] in window order (all B*Hs*Ws rows when rows is None)."""
    x = _c(x, np.float32)
    B, Hs, Ws, C = x.shape
    gamma = _c(gamma, np.float32); beta = _c(beta, np.float32)
    r = None if rows is None else _c(rows, np.int64)
    n = B * Hs * Ws if r is None else r.shape[0]
    out = np.empty((n, C), np.int8)
    yh = np.empty((n, C), np.float32) if return_yhat else None
    inv = np.float32(1.0) / np.float32(s_q)
    lib().oracle_op1(_p(x), B, Hs, Ws, C, int(M), int(shift), _p(gamma), _p(beta), float(eps), float(inv), int(z_q),
                     _p(r), n, _p(out), _p(yh))
    return (out, yh) if return_yhat else out


def qkv(X, W, s_w, b, s_x, z_x, s_q, s_k, s_v, return_acc=False):
    """QKV GEMM + fused op #2.  X int8 [T][C], W int8 [3C][C] -> int8 [T][3C]."""
    X = _c(X, np.int8); W = _c(W, np.int8); s_w = _c(s_w, np.float32); b = _c(b, np.float32)
    T, C = X.shape
    out = np.empty((T, 3 * C), np.int8)
    acc = np.empty((T, 3 * C), np.int32) if return_acc else None
    lib().oracle_qkv(_p(X), T, C, int(z_x), _p(W), _p(s_w), _p(b), float(s_x), float(s_q), float(s_k), float(s_v),
                     _p(acc), _p(out))
    return (out, acc) if return_acc else out


def rel_bias(table, M, heads):
    """Relative position bias [heads][N][N] from the [(2M-1)^2][heads] table (reading R24)."""
    table = _c(table, np.float32)
    N = M * M
    out = np.empty((heads, N, N), np.float32)
    lib().oracle_rel_bias(_p(table), int(M), int(heads), _p(out))
    return out


def shift_mask(Hs, Ws, M, shift):
    """Shifted-window mask [nW][N][N] of 0 / -100 (reading R25)."""
    N, nW = M * M, (Hs // M) * (Ws // M)
    out = np.empty((nW, N, N), np.float32)
    lib().oracle_shift_mask(int(Hs), int(Ws), int(M), int(shift), _p(out))
    return out


def attn_fold(s_q, s_k, s_v, s_a, D=32):
    """(m3, inv_p, m_o): op #3's dequant multiplier with the attention scale, the probability
    quantizer's reciprocal and the V.att requant multiplier (R23, R26, R27)."""
    o = np.empty(3, np.float32)
    lib().oracle_attn_fold(float(s_q), float(s_k), float(s_v), float(s_a), int(D), _p(o[0:]), _p(o[1:]), _p(o[2:]))
    return float(o[0]), float(o[1]), float(o[2])


def attn(qkv_q, A, B, wins=None, return_p=False):
    """Q.K GEMM -> fused op #3 -> V.att GEMM for the windows `wins` (all when None).  qkv_q: int8
    [B*Hs*Ws][3C] in window order; A: synth.AttnLayer.  Returns int8 [B*Hs*Ws][C] in raster order
    (rows of windows not computed are left 0) and, with return_p, Pq [nwins][heads][N][N]."""
    qkv_q = _c(qkv_q, np.int8)
    C, heads, M, Hs, Ws, s = A.C, A.heads, A.M, A.Hs, A.Ws, A.shift
    N = M * M
    n_win = qkv_q.shape[0] // N
    m3, inv_p, m_o = attn_fold(A.s_q, A.s_k, A.s_v, A.s_a, C // heads)
    bias = rel_bias(A.table, M, heads)
    mask = shift_mask(Hs, Ws, M, s) if s else None
    w = None if wins is None else _c(wins, np.int64)
    nw = n_win if w is None else w.shape[0]
    out = np.zeros((qkv_q.shape[0], C), np.int8)
    pt = np.empty((nw, heads, N, N), np.int8) if return_p else None
    lib().oracle_attn(_p(qkv_q), n_win, C, heads, M, Hs, Ws, int(s), float(m3), _p(bias), _p(mask), float(inv_p),
                      float(m_o), int(A.z_a), _p(w), nw, _p(out), _p(pt))
    return (out, pt) if return_p else out
