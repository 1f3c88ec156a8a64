"""Pins of the attention-half oracle (oracle/oracle_attn.c) against what the paper and the
mathematics fix -- never against itself (R21-R27).

  window geometry     torch.roll + reshape/permute (the Swin construction, a library path)
  op #1               closed forms of LayerNorm; float64 torch.layer_norm; shift 0 with one
                      window = raster order; the Q tie table
  op #2               brute-force integer dot products; power-of-two scales (every fp32 op
                      exact) with q / k / v thirds on their own scales
  rel. position bias  the Swin meshgrid construction; displacement-stationarity
  shift mask          the Swin img_mask slices; s = 0 -> no mask
  op #3 + V.att       uniform logits (p = 1/N exactly); one-hot logits; cross-region weight 0
                      under the mask; brute force in numpy float64 on tiny windows; the output
                      scatter is the inverse permutation of op #1's gather
"""
import numpy as np
import pytest
import torch

import oracle
import synth


# ---- window geometry (R21, R22) ---------------------------------------------------------------

def _swin_partition_order(B, Hs, Ws, M, s):
    """Raster row of every window-ordered row, by the Swin construction on an index tensor:
    torch.roll(x, (-s, -s), (1, 2)) then window_partition (view/permute/view)."""
    idx = torch.arange(B * Hs * Ws).view(B, Hs, Ws, 1)
    if s:
        idx = torch.roll(idx, shifts=(-s, -s), dims=(1, 2))
    w = idx.view(B, Hs // M, M, Ws // M, M, 1).permute(0, 1, 3, 2, 4, 5).contiguous().view(-1)
    return w.numpy()


@pytest.mark.parametrize("B,Hs,Ws,M,s", [(2, 4, 4, 2, 1), (1, 14, 14, 7, 3), (2, 12, 24, 12, 6), (1, 7, 7, 7, 0)])
def test_window_src_row_is_the_swin_roll_partition(B, Hs, Ws, M, s):
    ref = _swin_partition_order(B, Hs, Ws, M, s)
    got = np.array([oracle.window_src_row(r, Hs, Ws, M, s) for r in range(B * Hs * Ws)])
    np.testing.assert_array_equal(got, ref)
    assert sorted(got.tolist()) == list(range(B * Hs * Ws))   # a permutation


# ---- op #1 -------------------------------------------------------------------------------------

def _attn(C=64, Hs=4, Ws=4, M=2, shift=1, seed=5, **kw):
    return synth.make_attn_layer(C, Hs, Ws, seed, M=M, shift=shift, **kw)


def test_op1_constant_row_gives_beta():
    A = _attn()
    x = np.full((1, 4, 4, 64), 3.25, np.float32)
    out, yh = oracle.op1(x, A.gamma1, A.beta1, A.eps, A.s_x, A.z_x, A.M, A.shift, return_yhat=True)
    np.testing.assert_array_equal(yh, np.broadcast_to(A.beta1, yh.shape))
    np.testing.assert_array_equal(out, np.broadcast_to(oracle.quantize(A.beta1, A.s_x, 0), out.shape))


def test_op1_alternating_row_closed_form():
    """x = [a, -a, a, -a, ...]: mu = 0, var = a^2, yhat = +-a / sqrt(a^2 + eps) * gamma + beta."""
    A = _attn()
    a = 0.75
    row = np.tile(np.array([a, -a], np.float32), 32)
    x = np.broadcast_to(row, (1, 4, 4, 64)).copy()
    _, yh = oracle.op1(x, A.gamma1, A.beta1, A.eps, A.s_x, 0, A.M, A.shift, return_yhat=True)
    xh = np.where(np.arange(64) % 2 == 0, a, -a) / np.sqrt(a * a + A.eps)
    ref = (xh * A.gamma1.astype(np.float64) + A.beta1.astype(np.float64)).astype(np.float32)
    np.testing.assert_array_equal(yh[0], ref)


def test_op1_one_window_no_shift_is_raster_layer_norm():
    """shift 0 and M = Hs = Ws: window order == raster order, and yhat == float64 layer_norm."""
    A = _attn(C=96, Hs=7, Ws=7, M=7, shift=0)
    x = synth.make_block_input(2, 7, 7, 96, 3)
    out, yh = oracle.op1(x, A.gamma1, A.beta1, A.eps, A.s_x, A.z_x, 7, 0, return_yhat=True)
    ln = torch.nn.functional.layer_norm(torch.from_numpy(x).double().view(-1, 96), (96,),
                                        torch.from_numpy(A.gamma1).double(), torch.from_numpy(A.beta1).double(),
                                        eps=A.eps).float().numpy()
    np.testing.assert_allclose(yh, ln, rtol=0, atol=2e-6)
    np.testing.assert_array_equal(out, oracle.quantize(yh, A.s_x, A.z_x).reshape(out.shape))


def test_op1_shift_permutes_rows():
    """op #1 with a shift = op #1 without, rows permuted by the geometry (LN is per token)."""
    A = _attn(C=64, Hs=14, Ws=14, M=7, shift=3)
    x = synth.make_block_input(1, 14, 14, 64, 8)
    flat = oracle.op1(x, A.gamma1, A.beta1, A.eps, A.s_x, 0, 14, 0)          # one window, raster order
    got = oracle.op1(x, A.gamma1, A.beta1, A.eps, A.s_x, 0, 7, 3)
    np.testing.assert_array_equal(got, flat[_swin_partition_order(1, 14, 14, 7, 3)])


# ---- op #2 -------------------------------------------------------------------------------------

def test_qkv_brute_force_integer_dot():
    rng = np.random.default_rng(1)
    C, T = 32, 5
    X = rng.integers(-128, 128, (T, C)).astype(np.int8)
    W = rng.integers(-127, 128, (3 * C, C)).astype(np.int8)
    out, acc = oracle.qkv(X, W, np.ones(3 * C, np.float32), None, 1.0, -3, 1.0, 1.0, 1.0, return_acc=True)
    for t in range(T):
        for n in range(3 * C):
            assert acc[t, n] == sum((int(X[t, k]) + 3) * int(W[n, k]) for k in range(C))


def test_qkv_power_of_two_scales_exact_with_ties():
    """s_x = 2^-4, s_w = 2^-6, b = k/1024 -> y = A/1024 + b exactly; s_q/s_k/s_v = 2^-3/2^-2/2^-1
    -> out = rne(y * 8 / 4 / 2) on exact rationals (round-half-even on the ties)."""
    from fractions import Fraction
    rng = np.random.default_rng(2)
    C, T = 32, 7
    X = rng.integers(-20, 21, (T, C)).astype(np.int8)
    W = rng.integers(-20, 21, (3 * C, C)).astype(np.int8)
    b = (rng.integers(-64, 65, 3 * C) / 1024.0).astype(np.float32)
    out, acc = oracle.qkv(X, W, np.full(3 * C, 2.0 ** -6, np.float32), b, 2.0 ** -4, 0, 2.0 ** -3, 2.0 ** -2,
                          2.0 ** -1, return_acc=True)
    ties = 0
    for t in range(T):
        for n in range(3 * C):
            y = Fraction(int(acc[t, n]), 1024) + Fraction(float(b[n]))
            v = y * (8, 4, 2)[n // C]
            q = max(-128, min(127, round(v)))            # Python round: half to even
            ties += v.denominator == 2
            assert out[t, n] == q, (t, n, v)
    assert ties > 0


# ---- relative position bias and mask ------------------------------------------------------------

def _swin_rel_index(M):
    coords = torch.stack(torch.meshgrid(torch.arange(M), torch.arange(M), indexing="ij")).flatten(1)
    rel = (coords[:, :, None] - coords[:, None, :]).permute(1, 2, 0).contiguous()
    rel[:, :, 0] += M - 1
    rel[:, :, 1] += M - 1
    rel[:, :, 0] *= 2 * M - 1
    return rel.sum(-1).numpy()


@pytest.mark.parametrize("M,heads", [(2, 3), (7, 3), (12, 2)])
def test_rel_bias_is_the_swin_index(M, heads):
    rng = np.random.default_rng(M)
    table = rng.standard_normal(((2 * M - 1) ** 2, heads)).astype(np.float32)
    got = oracle.rel_bias(table, M, heads)
    idx = _swin_rel_index(M)
    for h in range(heads):
        np.testing.assert_array_equal(got[h], table[idx, h])
    # displacement-stationary: equal (dy, dx) -> equal bias; the diagonal is the centre entry
    c = (M - 1) * (2 * M - 1) + (M - 1)
    np.testing.assert_array_equal(np.diagonal(got, axis1=1, axis2=2), np.repeat(table[c][:, None], M * M, 1))


@pytest.mark.parametrize("Hs,Ws,M,s", [(4, 4, 4, 2), (14, 14, 7, 3), (24, 12, 12, 6)])
def test_shift_mask_is_the_swin_img_mask(Hs, Ws, M, s):
    img = np.zeros((Hs, Ws), np.int64)
    cnt = 0
    for hs in (slice(0, -M), slice(-M, -s), slice(-s, None)):
        for ws in (slice(0, -M), slice(-M, -s), slice(-s, None)):
            img[hs, ws] = cnt
            cnt += 1
    win = img.reshape(Hs // M, M, Ws // M, M).transpose(0, 2, 1, 3).reshape(-1, M * M)
    ref = np.where(win[:, :, None] == win[:, None, :], 0.0, -100.0).astype(np.float32)
    np.testing.assert_array_equal(oracle.shift_mask(Hs, Ws, M, s), ref)
    assert not oracle.shift_mask(Hs, Ws, M, 0).any()


# ---- op #3 and V.att ----------------------------------------------------------------------------

def test_attn_fold_power_of_two():
    m3, inv_p, m_o = oracle.attn_fold(2.0 ** -3, 2.0 ** -4, 2.0 ** -2, 2.0 ** -5, D=16)
    assert m3 == 2.0 ** -9 and inv_p == np.float32(1.0) / np.float32(np.float32(1.0) / np.float32(127.0))
    assert m_o == np.float32(np.float32(np.float32(1.0 / 127.0) * np.float32(0.25)) * np.float32(32.0))


def _qkv_from(q, k, v):
    return np.concatenate([q, k, v], axis=1).astype(np.int8)


def test_attn_uniform_logits_give_one_over_n():
    """q = 0, zero bias, no mask: every logit is 0, p = 1/N exactly, Pq = rne(127/N)."""
    A = _attn(C=64, Hs=14, Ws=14, M=7, shift=0)
    A.table = np.zeros_like(A.table)
    rng = np.random.default_rng(3)
    T = 196
    v = rng.integers(-60, 61, (T, 64)).astype(np.int8)
    qkv = _qkv_from(np.zeros((T, 64)), rng.integers(-127, 128, (T, 64)), v)
    out, P = oracle.attn(qkv, A, 1, return_p=True)
    assert (P == round(127 / 49)).all()
    m3, inv_p, m_o = oracle.attn_fold(A.s_q, A.s_k, A.s_v, A.s_a, 32)
    order = _swin_partition_order(1, 14, 14, 7, 0)
    for w in range(4):
        rows = np.arange(w * 49, (w + 1) * 49)
        O = 3 * v[rows].astype(np.int64).sum(0)            # every row of the window: the same
        ref = oracle.quantize((O.astype(np.float32) * np.float32(m_o)), 1.0, A.z_a)
        for i in rows:
            np.testing.assert_array_equal(out[order[i]], ref)


def test_attn_one_hot_logits():
    """k[j*] aligned with q and much larger than every other key: Pq[i][j*] = 127, the rest 0,
    so the output row is Q(fl(fl(127 * v[j*]) * m_o))."""
    A = _attn(C=32, Hs=7, Ws=7, M=7, shift=0)
    A.table = np.zeros_like(A.table)
    T = 49
    q = np.full((T, 32), 100, np.int8)
    k = np.zeros((T, 32), np.int8)
    k[11] = 100
    v = np.random.default_rng(4).integers(-127, 128, (T, 32)).astype(np.int8)
    out, P = oracle.attn(_qkv_from(q, k, v), A, 1, return_p=True)
    assert (P[0, 0, :, 11] == 127).all() and (np.delete(P[0, 0], 11, axis=1) == 0).all()
    _, _, m_o = oracle.attn_fold(A.s_q, A.s_k, A.s_v, A.s_a, 32)
    ref = oracle.quantize((127 * v[11].astype(np.int64)).astype(np.float32) * np.float32(m_o), 1.0, A.z_a)
    np.testing.assert_array_equal(out, np.broadcast_to(ref, out.shape))


def test_attn_shift_mask_zeroes_cross_region_weight():
    A = _attn(C=64, Hs=14, Ws=14, M=7, shift=3)
    rng = np.random.default_rng(6)
    qkv = rng.integers(-40, 41, (196, 192)).astype(np.int8)
    _, P = oracle.attn(qkv, A, 1, return_p=True)
    mask = oracle.shift_mask(14, 14, 7, 3)
    for w in range(4):
        cross = mask[w] < 0
        assert (P[w][:, cross] == 0).all()
        if w == 3:
            assert cross.any()


def test_attn_brute_force_numpy_float64():
    """Tiny windows (M = 2, N = 4), two heads of 32: S, the softmax (numpy float64), Pq, the int
    V.att product and the requant, written independently and compared element by element."""
    A = _attn(C=64, Hs=4, Ws=4, M=2, shift=1, seed=9)
    rng = np.random.default_rng(10)
    T = 16
    qkv = rng.integers(-127, 128, (T, 192)).astype(np.int8)
    out, P = oracle.attn(qkv, A, 1, return_p=True)
    m3, inv_p, m_o = oracle.attn_fold(A.s_q, A.s_k, A.s_v, A.s_a, 32)
    bias = oracle.rel_bias(A.table, 2, 2)
    mask = oracle.shift_mask(4, 4, 2, 1)
    order = _swin_partition_order(1, 4, 4, 2, 1)
    f32 = np.float32
    for w in range(4):
        rows = np.arange(4 * w, 4 * w + 4)
        for h in range(2):
            q = qkv[rows, 32 * h:32 * h + 32].astype(np.int64)
            k = qkv[rows, 64 + 32 * h:64 + 32 * h + 32].astype(np.int64)
            v = qkv[rows, 128 + 32 * h:128 + 32 * h + 32].astype(np.int64)
            S = q @ k.T
            logit = ((S.astype(f32) * f32(m3)).astype(f32) + bias[h]).astype(f32)
            logit = (logit + mask[w]).astype(f32)
            e = np.exp(logit.astype(np.float64) - logit.max(1, keepdims=True))
            p = (e / e.sum(1, keepdims=True)).astype(f32)
            Pq = np.clip(np.rint((p * f32(inv_p)).astype(f32)), -128, 127).astype(np.int64)
            np.testing.assert_array_equal(P[w, h], Pq)
            O = Pq @ v
            ref = np.clip(np.rint((O.astype(f32) * f32(m_o)).astype(f32)) + A.z_a, -128, 127)
            np.testing.assert_array_equal(out[order[rows], 32 * h:32 * h + 32], ref)
