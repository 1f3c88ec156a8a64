"""Pins of the CPU oracle against what the paper and the mathematics fix
(not against the oracle itself).  -m "not gpu": runs in the CPU container.

Each pin names the oracle step and the PAPER.md
passage it follows.  A plausible slip anywhere in the oracle — a dropped
bias or zero-point term, a transposed weight, a wrong rounding mode, a
sign error in the LayerNorm — fails at least one test here.
"""
import itertools
import math
import os

import numpy as np
import pytest

import oracle
import synth
from conftest import load_table

RNG = np.random.default_rng(2402_01169)


# ---------------------------------------------------------------- O1 / O3
def _triple_loop(X, W, zp):
    """Pure-Python brute force (tiny shapes only): sum_k (x - zp) * w."""
    T, K = X.shape
    N = W.shape[0]
    out = [[0] * N for _ in range(T)]
    for t in range(T):
        for n in range(N):
            s = 0
            for k in range(K):
                s += (int(X[t, k]) - zp) * int(W[n, k])
            out[t][n] = s
    return np.array(out, dtype=np.int64)


@pytest.mark.parametrize("T,K,N,zp", [(1, 1, 1, 0), (3, 5, 7, 0), (8, 64, 256, 0), (5, 33, 17, -128),
                                      (4, 64, 96, -7), (2, 16, 8, 127)])
def test_gemm_bruteforce(T, K, N, zp):
    """O1: PAPER.md:225-226 (int8 weights x int8 activations on integer tensor cores)."""
    X = RNG.integers(-128, 128, (T, K), dtype=np.int8)
    W = RNG.integers(-127, 128, (N, K), dtype=np.int8)
    X[0, 0], W[0, 0] = -128, -127  # extremes
    ref = _triple_loop(X, W, zp)
    got = oracle.gemm_i8(X, W, zp)
    assert got.dtype == np.int32
    np.testing.assert_array_equal(got.astype(np.int64), ref)
    # library cross-check (int64 matmul), W is [N][K] so the product is X @ W^T
    lib = (X.astype(np.int64) - zp) @ W.astype(np.int64).T
    np.testing.assert_array_equal(got.astype(np.int64), lib)


def test_gemm_closed_forms():
    """O1 closed forms: X == z -> 0; (X - z) == 1 and W == 1 -> K; one-hot rows pick W columns."""
    K, N = 96, 40
    W = RNG.integers(-127, 128, (N, K), dtype=np.int8)
    for zp in (0, -7, -128):
        X = np.full((3, K), zp, np.int8)
        assert not oracle.gemm_i8(X, W, zp).any()
        X1 = np.full((2, K), zp + 1, np.int8)
        np.testing.assert_array_equal(oracle.gemm_i8(X1, np.ones((N, K), np.int8), zp), K)
    # one-hot: X[t] = z + e_j  -> A[t, n] = W[n, j]
    zp = -3
    X = np.full((K, K), zp, np.int8)
    X[np.arange(K), np.arange(K)] = zp + 1
    np.testing.assert_array_equal(oracle.gemm_i8(X, W, zp), W.T.astype(np.int32))
    # non-square: a transposed operand would change the shape or the values
    Xr = RNG.integers(-128, 128, (5, K), dtype=np.int8)
    assert oracle.gemm_i8(Xr, W, 0).shape == (5, N)


def test_gemm_extreme_and_overflow():
    """D2: |A| <= 255*127*K fits int32 for K <= 6144 (Swin-L FC2); a larger K overflows and is caught."""
    K = 6144
    X = np.full((1, K), 127, np.int8)
    W = np.full((2, K), -127, np.int8)
    A = oracle.gemm_i8(X, W, -128)            # (127+128) * -127 * K
    assert int(A[0, 0]) == 255 * -127 * K
    Kbig = 70000                              # 255*127*70000 > 2^31
    with pytest.raises(OverflowError):
        oracle.gemm_i8(np.full((1, Kbig), 127, np.int8), np.full((1, Kbig), 127, np.int8), -128)


def test_gemm_row_subset():
    """Rows are independent (Fig. 1: the MLP is token-wise): a row subset equals the same rows of the full result."""
    X = RNG.integers(-128, 128, (50, 32), dtype=np.int8)
    W = RNG.integers(-127, 128, (24, 32), dtype=np.int8)
    rows = np.array([49, 0, 7, 7, 13])
    np.testing.assert_array_equal(oracle.gemm_i8(X, W, 3, rows=rows), oracle.gemm_i8(X, W, 3)[rows])


# ---------------------------------------------------------------- Q / dQ
def test_q_tie_table(golden_dir):
    """PAPER.md:124 Q; round half to even (R2); saturation to [-128, 127] (R6)."""
    for x, z, exp in load_table(os.path.join(golden_dir, "q_ties.txt")):
        got = oracle.quantize(np.float32(float(x)), 1.0, int(z))[0]
        assert int(got) == int(exp), (x, z, exp, got)


def test_q_spec_example_under_rne():
    """SPEC.md:80's edge: Q(0.005, s=0.01).  fl(0.005f * fl(1/0.01f)) == 0.5 exactly,
    so round-half-to-even gives 0 (SPEC's half-away-from-zero would give 1)."""
    assert np.float32(0.005) * (np.float32(1) / np.float32(0.01)) == np.float32(0.5)
    assert int(oracle.quantize(0.005, 0.01, 0)[0]) == 0
    assert int(oracle.quantize(0.015, 0.01, 0)[0]) == 2   # 1.5 -> 2 under either rule? 0.015f*100 -> 1.5 -> 2


def test_grid_round_trip_exhaustive():
    """O6 invariant: Q(dQ(q)) == q for every q in [-128, 127], random (s, z).
    Error of dQ then Q is <= 255 * 2^-23 << 0.5, so the grid value is recovered."""
    q = np.arange(-128, 128, dtype=np.int8)
    rng = np.random.default_rng(7)
    for _ in range(200):
        s = float(np.float32(10 ** rng.uniform(-6, 2)))
        z = int(rng.integers(-128, 128))
        qq = np.arange(-128, 128)
        x = oracle.dequantize(q, s, z)
        back = oracle.quantize(x, s, z)
        # values whose (q - z) overflows the grid only saturate; q itself is always in range
        np.testing.assert_array_equal(back.astype(np.int32), qq)


def test_round_trip_bound():
    """|x - dQ(Q(x))| <= s/2 for |x| <= 127 s (plus fp32 rounding of x*(1/s))."""
    s = np.float32(1 / 127)
    x = np.random.default_rng(3).uniform(-1, 1, 10000).astype(np.float32)
    err = np.abs(x - oracle.dequantize(oracle.quantize(x, s, 0), s, 0))
    assert err.max() <= s / 2 * (1 + 1e-5)


# ---------------------------------------------------------------- O0
def test_fold_constants_definition():
    """O0: m1 = fl(s_x*s_w1), inv_h = fl(1/s_h), m2 = fl(s_h*s_w2), inv_y = fl(1/s_y)
    (IEEE fp32, one rounding each; numpy float32 arithmetic is IEEE-correct)."""
    s_w1 = np.float32(10.0) ** RNG.uniform(-5, -1, 64).astype(np.float32)
    s_w2 = np.float32(10.0) ** RNG.uniform(-5, -1, 16).astype(np.float32)
    m1, ih, m2, iy = oracle.fold_constants(0.0123, s_w1, 0.0457, s_w2, 0.039)
    np.testing.assert_array_equal(m1, np.float32(0.0123) * s_w1)
    np.testing.assert_array_equal(m2, np.float32(0.0457) * s_w2)
    assert np.float32(ih) == np.float32(1) / np.float32(0.0457)
    assert np.float32(iy) == np.float32(1) / np.float32(0.039)
    # exact when the scales are powers of two
    m1, ih, _, _ = oracle.fold_constants(2.0 ** -4, np.full(4, 2.0 ** -6, np.float32), 2.0 ** -7,
                                         np.ones(2, np.float32), 1.0)
    assert (m1 == 2.0 ** -10).all() and ih == 128.0


# ---------------------------------------------------------------- O2
def test_ep5_pow2_table(golden_dir):
    """O2 with exact power-of-two scales against the hand-computed table."""
    rows = load_table(os.path.join(golden_dir, "ep5_pow2_table.txt"))
    for a1, b1k, zh, exp in rows:
        A1 = np.array([[int(a1)]], np.int32)
        b1 = np.array([int(b1k) / 1024.0], np.float32) if int(b1k) else None
        got = oracle.ep5(A1, np.array([2.0 ** -10], np.float32), b1, 128.0, int(zh))
        assert int(got[0, 0]) == int(exp), (a1, b1k, zh, exp, int(got[0, 0]))


def _linear_q(y, inv_h, z_h):
    # Q of the un-activated value: clamp(rne(fl(y*inv_h)) + z_h) (numpy fp32 mult is IEEE)
    v = (y.astype(np.float32) * np.float32(inv_h)).astype(np.float32)
    return np.clip(np.rint(v.astype(np.float64)) + z_h, -128, 127).astype(np.int8)


@pytest.mark.parametrize("z_h", [0, -128, -7])
def test_ep5_relu_is_clamp_at_zero_point(z_h):
    """Invariant: quantized ReLU == max(quantized identity, z_h) elementwise, exactly.
    Holds because rne is monotone and rne(0) = 0 — the reason ReLU can be applied in the integer
    domain after the GEMM."""
    A1 = RNG.integers(-3_000_000, 3_000_000, (64, 96), dtype=np.int32)
    m1 = (RNG.uniform(0.5, 2, 96) * 1e-5).astype(np.float32)
    b1 = (RNG.standard_normal(96) * 0.02).astype(np.float32)
    inv_h = float(np.float32(1) / np.float32(0.37 / 127))
    Hq, pre = oracle.ep5(A1, m1, b1, inv_h, z_h, return_pre=True)
    # pre = fmaf(fl(A1), m1, b1): check it against an exact rational evaluation rounded once
    a = A1.astype(np.float32).astype(np.float64)
    exact = a * m1.astype(np.float64) + b1.astype(np.float64)  # exact in double? products < 2^53: yes (24+24 bits)
    np.testing.assert_array_equal(pre, exact.astype(np.float32))
    lin = _linear_q(pre, inv_h, z_h)
    np.testing.assert_array_equal(Hq, np.maximum(lin, np.int8(z_h)))


def test_ep5_relu_scale_commutation():
    """PAPER.md:139 vs ReLU: max(y,0)*s == max(y*s, 0) bitwise for s > 0."""
    y = RNG.standard_normal(100000).astype(np.float32)
    for s in (np.float32(0.37), np.float32(1 / 3), np.float32(1e-3), np.float32(77.0)):
        np.testing.assert_array_equal(np.maximum(y, 0) * s, np.maximum(y * s, 0))


def test_ep5_relu_on_int32_accumulator():
    """With b1 = NULL (the paper's GELU-less block), ReLU on the int32 accumulator
    before dequantization gives bit-identical Hq ("fused, as an integer operation")."""
    A1 = RNG.integers(-2_000_000, 2_000_000, (32, 128), dtype=np.int32)
    m1 = (RNG.uniform(0.5, 2, 128) * 1e-5).astype(np.float32)
    inv_h = 127 / 0.5
    a = oracle.ep5(A1, m1, None, inv_h, 0)
    b = oracle.ep5(np.maximum(A1, 0), m1, None, inv_h, 0)
    np.testing.assert_array_equal(a, b)


def test_ep5_gelu_library_and_closed_forms():
    """O2' (GELU control): m1 = 1 (y = A1 exactly), inv_h = 64 (s_h = 2^-6).
    Closed forms gelu(0)=0, gelu(1)=0.8413447, gelu(-2)=-0.0455003, gelu(10)=10,
    and a float64 library cross-check over a sweep (torch GELU, approximate='none')."""
    import torch
    A1 = np.array([[0, 1, -2, 10, -1, 3]], np.int32)
    got = oracle.ep5(A1, np.ones(6, np.float32), None, 64.0, 0, act=oracle.ACT_GELU)
    want = [0, round(64 * 0.8413447), round(64 * -0.0455003), 127, round(64 * -0.1586553), 127]
    assert got[0].tolist() == want
    # library sweep: y = A1 * m with m = 2^-12 (exact), v = fl(fl(gelu(y)) * 32)
    A = np.arange(-40000, 40000, 7, dtype=np.int32)[None, :]
    m = np.full(A.shape[1], 2.0 ** -12, np.float32)
    got = oracle.ep5(A, m, None, 32.0, 0, act=oracle.ACT_GELU)[0]
    y = torch.tensor(A[0].astype(np.float64) * 2.0 ** -12)
    g = torch.nn.functional.gelu(y, approximate="none").numpy().astype(np.float32)
    v = (g * np.float32(32.0)).astype(np.float64)
    ref = np.clip(np.rint(v), -128, 127).astype(np.int8)
    assert (got != ref).sum() == 0
    # the non-linearity obstruction of PAPER.md:139 (f(s x) != s f(x)), witness s=2, x=-1
    gl = lambda x: 0.5 * x * (1 + math.erf(x / math.sqrt(2)))
    assert abs(gl(-2.0) - 2 * gl(-1.0)) > 1e-3


# ---------------------------------------------------------------- O4..O6
def _ep6(A2, m2, b2, X, s_x=1.0, z_x=0, gamma=None, beta=None, eps=1e-5, inv_y=1.0, z_y=0, R=None):
    C = A2.shape[1]
    gamma = np.ones(C, np.float32) if gamma is None else gamma
    beta = np.zeros(C, np.float32) if beta is None else beta
    return oracle.ep6(A2, m2, b2, X, s_x, z_x, gamma, beta, eps, inv_y, z_y, R=R)


def test_ep6_residual_and_bias_terms():
    """O4 (PAPER.md:82-86 dQ -> FC2 bias -> Add): with A2 = 0 and R = 0, z == b2;
    with A2 = 0, b2 = 0, no R: z == dQ(X) = fl((X - z_x) * s_x) exactly (power-of-two s_x);
    with power-of-two m2: z = A2*m2 + b2 + r exactly."""
    C = 64
    A2 = np.zeros((3, C), np.int32)
    b2 = (RNG.standard_normal(C) * 0.02).astype(np.float32)
    X = RNG.integers(-128, 128, (3, C), dtype=np.int8)
    _, _, z = _ep6(A2, np.ones(C, np.float32), b2, X, R=np.zeros((3, C), np.float32))
    np.testing.assert_array_equal(z, np.broadcast_to(b2, (3, C)))
    _, _, z = _ep6(A2, np.ones(C, np.float32), None, X, s_x=2.0 ** -5, z_x=-7)
    np.testing.assert_array_equal(z, (X.astype(np.float64) + 7) * 2.0 ** -5)
    A2 = RNG.integers(-100000, 100000, (3, C), dtype=np.int32)
    b2 = (RNG.integers(-64, 64, C) * 2.0 ** -8).astype(np.float32)
    _, _, z = _ep6(A2, np.full(C, 2.0 ** -12, np.float32), b2, X, s_x=2.0 ** -6, z_x=3)
    exact = A2 * 2.0 ** -12 + b2.astype(np.float64) + (X.astype(np.float64) - 3) * 2.0 ** -6
    np.testing.assert_array_equal(z.astype(np.float64), exact)


def test_ln_closed_forms():
    """O5 (LayerNorm; biased variance): constant row -> yhat == beta exactly;
    two-element row [a, -a] -> +-a/sqrt(a^2+eps); gamma=1, beta=0: mean(xhat) ~ 0 and
    mean(xhat^2) == var/(var+eps)."""
    C = 96
    beta = (RNG.standard_normal(C) * 0.1).astype(np.float32)
    gamma = (1 + 0.1 * RNG.standard_normal(C)).astype(np.float32)
    R = np.full((2, C), 0.75, np.float32)
    _, yh, _ = _ep6(np.zeros((2, C), np.int32), np.ones(C, np.float32), None,
                    np.zeros((2, C), np.int8), gamma=gamma, beta=beta, R=R)
    np.testing.assert_array_equal(yh, np.broadcast_to(beta, (2, C)))
    a = 0.3
    _, yh, _ = _ep6(np.zeros((1, 2), np.int32), np.ones(2, np.float32), None,
                    np.zeros((1, 2), np.int8), R=np.array([[a, -a]], np.float32), eps=1e-5)
    want = np.float32(a) / math.sqrt(np.float32(a) ** 2 + np.float32(1e-5))
    np.testing.assert_allclose(yh[0], [want, -want], rtol=2e-7)
    R = (RNG.standard_normal((50, C)) * 3 + 1).astype(np.float32)
    _, yh, z = _ep6(np.zeros((50, C), np.int32), np.ones(C, np.float32), None,
                    np.zeros((50, C), np.int8), R=R, eps=1e-5)
    zd = z.astype(np.float64)
    var = zd.var(axis=1)
    assert np.abs(yh.astype(np.float64).mean(axis=1)).max() < 1e-6
    np.testing.assert_allclose((yh.astype(np.float64) ** 2).mean(axis=1), var / (var + 1e-5), rtol=1e-6)


def test_ln_library_cross_check():
    """O5 vs torch.nn.functional.layer_norm in float64 on the oracle's own z (rounded once to fp32)."""
    import torch
    C = 192
    R = (RNG.standard_normal((64, C)) * 2).astype(np.float32)
    gamma = (1 + 0.1 * RNG.standard_normal(C)).astype(np.float32)
    beta = (0.1 * RNG.standard_normal(C)).astype(np.float32)
    A2 = RNG.integers(-50000, 50000, (64, C), dtype=np.int32)
    m2 = (RNG.uniform(0.5, 2, C) * 1e-5).astype(np.float32)
    Y, yh, z = _ep6(A2, m2, None, np.zeros((64, C), np.int8), gamma=gamma, beta=beta, R=R,
                    inv_y=float(np.float32(127 / 5)))
    ref = torch.nn.functional.layer_norm(torch.tensor(z, dtype=torch.float64), (C,),
                                         torch.tensor(gamma, dtype=torch.float64),
                                         torch.tensor(beta, dtype=torch.float64), eps=1e-5).numpy()
    np.testing.assert_allclose(yh, ref.astype(np.float32), rtol=0, atol=2e-6)
    v = (yh * np.float32(127 / 5)).astype(np.float64)
    np.testing.assert_array_equal(Y, np.clip(np.rint(v), -128, 127).astype(np.int8))


# ---------------------------------------------------------------- O7
def test_layer_composition_and_taps():
    """O7 = O1 -> O2 -> O3 -> O4..O6: the composed layer equals the staged steps."""
    L = synth.make_layer(64, 11, fc1_bias=True, z_x=-5, z_h=-128, z_y=3)
    X = synth.make_activations(L, 37, 12)
    taps = oracle.mlp(L, X, taps=True)
    m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
    a1 = oracle.gemm_i8(X, L.w1, L.z_x)
    h = oracle.ep5(a1, m1, L.b1, ih, L.z_h)
    a2 = oracle.gemm_i8(h, L.w2, L.z_h)
    Y, yh, z = oracle.ep6(a2, m2, L.b2, X, L.s_x, L.z_x, L.gamma, L.beta, L.eps, iy, L.z_y)
    for k, v in (("acc1", a1), ("hidden", h), ("acc2", a2), ("yhat", yh), ("z", z), ("y", Y)):
        np.testing.assert_array_equal(taps[k], v, err_msg=k)
    rows = np.array([36, 0, 5])
    np.testing.assert_array_equal(oracle.mlp(L, X, rows=rows), Y[rows])


@pytest.mark.parametrize("C,act,bias", [(96, 0, False), (128, 0, True), (96, 1, True)])
def test_layer_float_reference_budget(C, act, bias):
    """O7 sanity (parity-unpinned by the paper: it prints no per-layer values): the int8 layer
    tracks a float64 dequantize-everything MLP (ReLU/GELU, LayerNorm) within the quantization
    budget.  A transposed weight, a dropped bias or residual, or a wrong LN shifts this by far
    more than the budget."""
    import torch
    L = synth.make_layer(C, 100 + C, act=act, fc1_bias=bias)
    X = synth.make_activations(L, 256, 7)
    Y = oracle.mlp(L, X).astype(np.float64)
    x = (X.astype(np.float64) - L.z_x) * L.s_x
    w1 = L.w1.astype(np.float64) * L.s_w1[:, None]
    w2 = L.w2.astype(np.float64) * L.s_w2[:, None]
    y1 = x @ w1.T + (L.b1 if L.b1 is not None else 0)
    t1 = torch.tensor(y1)
    h = (torch.relu(t1) if act == 0 else torch.nn.functional.gelu(t1)).numpy()
    y2 = h @ w2.T + L.b2 + x
    ln = torch.nn.functional.layer_norm(torch.tensor(y2), (C,), torch.tensor(L.gamma, dtype=torch.float64),
                                        torch.tensor(L.beta, dtype=torch.float64), eps=L.eps).numpy()
    Yf = np.clip(np.rint(ln / L.s_y) + L.z_y, -128, 127)
    d = np.abs(Y - Yf)
    assert np.mean(d <= 2) > 0.995, np.mean(d <= 2)
    assert np.abs(np.mean(Y - Yf)) < 0.2


def test_recipe_non_degenerate():
    """DESIGN.md §4 input recipe: ReLU zero fraction 40-60 %, hidden saturation < 1 %,
    output saturation < 1 %, no all-zero rows (random data, not zeros)."""
    for C in (96, 192, 384):
        L = synth.make_layer(C, synth.layer_seed(2, 0, C), act=0)
        X = synth.make_activations(L, 512, 5)
        t = oracle.mlp(L, X, taps=True)
        h = t["hidden"]
        assert 0.40 <= (h == L.z_h).mean() <= 0.60
        assert (h == 127).mean() < 0.01
        assert (np.abs(t["y"].astype(int)) >= 127).mean() < 0.01
        assert (np.abs(X.astype(int)).sum(1) > 0).all()


def test_ep6_residual_dq_then_add():
    """Reading R3 / Fig. 1 (dQ -> FC2 Bias -> Add, each node its own step): with
    residual == NULL the residual is dQ(X) = fl(fl(X - z_x) * s_x) (the dQ of PAPER.md:124) and
    z = fl(d + dQ(X)) -- two roundings, pinned against exact rational arithmetic (each rounding
    done on the exact rational value, not by another float formula)."""
    from fractions import Fraction

    def f32(q):   # exact round-to-nearest-even of a rational to float32
        c = np.float32(float(q))
        cands = [np.nextafter(c, np.float32(-np.inf)), c, np.nextafter(c, np.float32(np.inf))]
        return min(cands, key=lambda v: (abs(Fraction(float(v)) - q), int(np.float32(v).view(np.uint32)) & 1))

    rng = np.random.default_rng(11)
    C = 64
    A2 = rng.integers(-20000, 20000, size=(4, C)).astype(np.int32)
    m2 = (rng.random(C).astype(np.float32) * np.float32(1e-4)).astype(np.float32)
    b2 = (rng.standard_normal(C) * 0.02).astype(np.float32)
    X = rng.integers(-128, 128, size=(4, C)).astype(np.int8)
    s_x, z_x = np.float32(0.2125984), 3
    _, _, z = _ep6(A2, m2, b2, X, s_x=float(s_x), z_x=z_x)
    differs = 0
    for t in range(4):
        for c in range(C):
            d = f32(Fraction(float(np.float32(A2[t, c]))) * Fraction(float(m2[c])) +
                    Fraction(float(b2[c])))                         # fmaf(fl(A2), m2, b2)
            r = f32(Fraction(int(X[t, c]) - z_x) * Fraction(float(s_x)))   # dQ(X)
            assert z[t, c] == f32(Fraction(float(d)) + Fraction(float(r))), (t, c)
            one = f32(Fraction(int(X[t, c]) - z_x) * Fraction(float(s_x)) + Fraction(float(d)))
            differs += one != z[t, c]
    assert differs > 0   # the case actually distinguishes two roundings from one (an fma)


# ---------------------------------------------------------------- NEXT-2: proj GEMM + op #4 (+ LN2)
def test_proj_op4_pins():
    """oracle.proj_op4 (Fig. 1 lines 63-70; R18): (i) A is the brute-force
    integer product with the input zero point; (ii) power-of-two scales make every fp32 op exact:
    z == A * s_a * s_w + b + R in float64; (iii) yhat == torch float64 layer_norm(z) (LN2),
    Y == clamp(rne(fl(yhat * 1/s_y)) + z_y); (iv) W = 0 and a constant shortcut row give
    yhat == beta exactly (the bias and the residual enter once, before LN2)."""
    import torch
    C, T = 64, 9
    P = synth.make_proj(C, 31, z_a=-3, z_y=2)
    P.s_a = 2.0 ** -4
    P.s_w = np.full(C, 2.0 ** -6, np.float32)
    P.b = (RNG.integers(-64, 64, C) * 2.0 ** -10).astype(np.float32)
    P.s_y = 2.0 ** -5
    A_in = RNG.integers(-128, 128, (T, C), dtype=np.int8)
    R = (RNG.integers(-4096, 4096, (T, C)) * 2.0 ** -10).astype(np.float32)
    Y, yh, z, A = oracle.proj_op4(P, A_in, R)
    np.testing.assert_array_equal(A, _triple_loop(A_in, P.w, -3))
    exact = A.astype(np.float64) * 2.0 ** -10 + P.b.astype(np.float64) + R.astype(np.float64)
    np.testing.assert_array_equal(z.astype(np.float64), exact)
    ref = torch.nn.functional.layer_norm(torch.tensor(z, dtype=torch.float64), (C,),
                                         torch.tensor(P.gamma, dtype=torch.float64),
                                         torch.tensor(P.beta, dtype=torch.float64), eps=P.eps).numpy()
    np.testing.assert_allclose(yh, ref.astype(np.float32), rtol=0, atol=2e-6)
    v = (yh * np.float32(32.0)).astype(np.float64)
    np.testing.assert_array_equal(Y, np.clip(np.rint(v) + 2, -128, 127).astype(np.int8))
    P.w = np.zeros((C, C), np.int8)
    P.b = None
    Rc = np.full((3, C), 1.25, np.float32)
    _, yh, z, A = oracle.proj_op4(P, A_in[:3], Rc)
    assert (A == 0).all()
    np.testing.assert_array_equal(z, Rc)
    np.testing.assert_array_equal(yh, np.broadcast_to(P.gamma * 0 + P.beta, (3, C)))


# ---- O2'': the I-ViT shift-GELU control (reading R28) -----------

def _sg_layer():
    import synth
    return synth.make_layer(96, 5150, act=2)


def _sg_run(L, y_row, extra=None):
    """Hq of one row of pre-activations y (A1 built so fl(A1) * m1 = y exactly: m1 = 2^-10)."""
    y = np.asarray(y_row, np.float64)
    A1 = np.rint(y * 1024.0).astype(np.int32)[None, :]
    m1 = np.full(A1.shape[1], 2.0 ** -10, np.float32)
    inv_h = np.float32(1.0) / np.float32(L.s_h)
    Hq, I = oracle.ep5_shiftgelu(A1, m1, None, L.s_g, inv_h, 0, return_I=True)
    return Hq[0], I[0], A1[0] / 1024.0


def test_shiftgelu_zero_argument_is_exactly_one():
    """ShiftExp(0) = 2|x0| 2^14 and, with e_m ~ 0 (a large row max), sig = 127 or 128 at the max:
    the max element passes through (Hq = rne(y / s_h) within 1 LSB)."""
    L = _sg_layer()
    sig = 0.02 * np.sqrt(96 * 1.7)
    y = np.linspace(-2, 2, 384) * sig
    y[17] = 7.0 * sig                                     # the row max
    Hq, I, yq = _sg_run(L, y)
    assert I.max() == I[17]
    assert abs(int(Hq[17]) - int(np.clip(np.rint(yq[17] / L.s_h), -128, 127))) <= 1


def test_shiftgelu_matches_x_sigmoid_1p702x():
    """The shift approximations (x log2 e by shifts, 2^f ~ 1 + f/2 on f in (-1, 0]) stay within 7 %
    of x * sigmoid(1.702 x) -- the form I-ViT approximates -- plus 2 quantization steps; a sign
    or index error (wrong max, wrong operand) fails by tens of steps."""
    L = _sg_layer()
    sig = 0.02 * np.sqrt(96 * 1.7)
    y = np.linspace(-6, 6, 384) * sig
    Hq, I, yq = _sg_run(L, y)
    x = I.astype(np.float64) * L.s_g
    ref = x / (1.0 + np.exp(-1.702 * x)) / L.s_h
    tol = 0.07 * np.abs(x) / L.s_h + 2.0
    assert (np.abs(Hq - np.clip(ref, -128, 127)) <= tol).all(), np.abs(Hq - ref).max()
    assert (np.diff(Hq[y > 0].astype(int)) >= -1).all()   # monotone right of 0 (up to rounding)


def test_shiftgelu_depends_on_the_row_max_only_through_rounding():
    """sigmoid(1.702 x) = e^{S(I-Im)} / (e^{S(I-Im)} + e^{-S Im}) for any Im: raising the row max
    (another element) may move outputs by the integer approximations' rounding only."""
    L = _sg_layer()
    sig = 0.02 * np.sqrt(96 * 1.7)
    y = np.linspace(-3, 3, 384) * sig
    y2 = y.copy()
    y2[0] = 7.5 * sig                                     # a new, larger row max elsewhere
    Hq1, _, _ = _sg_run(L, y)
    Hq2, _, _ = _sg_run(L, y2)
    d = np.abs(Hq1[1:].astype(int) - Hq2[1:].astype(int))
    assert d.max() <= 1 and (d > 0).mean() < 0.5
