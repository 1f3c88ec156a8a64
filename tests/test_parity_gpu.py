"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle
on the same seeded inputs (synth/).  Run on a B200 with -m gpu.

Tiers (BASELINE.json north_star):
  acc1, acc2 (int32)                      bit-exact
  Hq, ReLU, canonical fp32 order          bit-exact
  Hq, GELU control                        <= 1 LSB on <= 0.01 % of elements
  Y (int8)                                <= 1 LSB on <= 0.01 % of elements
  yhat (pre-quant LayerNorm, fp32)        |gpu - ref| <= 1e-5 * max(1, |ref|)
Each stage is checked on the GPU's own input to that stage (oracle step
applied to the previous GPU tap), plus end to end against oracle.mlp.
"""
import numpy as np
import pytest

import oracle
import synth

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module")
def dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2402_01169_b200 as P
    P.lib()  # fails loudly if the extension is missing
    return torch.device("cuda:0")


def _layer(C, seed, act=0, bias=False, zx=0, zh=0, zy=0):
    return synth.make_layer(C, seed, act=act, fc1_bias=bias, z_x=zx, z_h=zh, z_y=zy)


def _tier_int8(got, ref, frac=1e-4, what=""):
    d = np.abs(got.astype(np.int32) - ref.astype(np.int32))
    assert d.max(initial=0) <= 1, f"{what}: max |diff| {d.max()} > 1 LSB"
    n_bad = int((d > 0).sum())
    assert n_bad <= max(0, int(frac * d.size)), f"{what}: {n_bad} of {d.size} elements differ (> {frac:%})"
    return n_bad


def _tier_yhat(got, ref, what="yhat"):
    err = np.abs(got.astype(np.float64) - ref.astype(np.float64))
    tol = 1e-5 * np.maximum(1.0, np.abs(ref.astype(np.float64)))
    assert (err <= tol).all(), f"{what}: max rel err {(err / tol).max() * 1e-5:.3e}"


def _run_and_check(dev, L, T, x_seed=5, resid=False, e2e=True, ln_fp64=False, op5_unfused=False):
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    X = synth.make_activations(L, T, x_seed)
    R = synth.make_residual(T, L.C, x_seed + 1) if resid else None
    layer = SwinMlpInt8Layer(L, device=0, ln_fp64=ln_fp64, op5_unfused=op5_unfused)
    xd = torch.from_numpy(X).to(dev)
    rd = torch.from_numpy(R).to(dev) if resid else None
    zo = torch.empty((T, L.C), dtype=torch.float32, device=dev)
    taps = layer.run_debug(xd, residual=rd, residual_out=zo)
    torch.cuda.synchronize()
    g = {k: v.cpu().numpy() for k, v in taps.items()}
    g["z"] = zo.cpu().numpy()
    # stage-wise
    m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
    a1 = oracle.gemm_i8(X, L.w1, L.z_x, nthreads=0)
    np.testing.assert_array_equal(g["acc1"], a1, err_msg="acc1 (FC1 int32) not bit-exact")
    if L.act == synth.ACT_SHIFT_GELU:
        h = oracle.ep5_shiftgelu(g["acc1"], m1, L.b1, L.s_g, ih, L.z_h)
    else:
        h = oracle.ep5(g["acc1"], m1, L.b1, ih, L.z_h, act=L.act)
    if L.act in (synth.ACT_RELU, synth.ACT_SHIFT_GELU):   # (shift-GELU: integer after two fp32 products)
        np.testing.assert_array_equal(g["hidden"], h, err_msg="Hq (ReLU / shift-GELU) not bit-exact")
    else:
        _tier_int8(g["hidden"], h, what="Hq (GELU)")
    a2 = oracle.gemm_i8(g["hidden"], L.w2, L.z_h)
    np.testing.assert_array_equal(g["acc2"], a2, err_msg="acc2 (FC2 int32) not bit-exact")
    Y, yh, z = oracle.ep6(g["acc2"], m2, L.b2, X, L.s_x, L.z_x, L.gamma, L.beta, L.eps, iy, L.z_y, R=R)
    np.testing.assert_array_equal(g["z"], z, err_msg="z (pre-LN sum) not bit-exact")
    _tier_yhat(g["yhat"], yh)
    flips = _tier_int8(g["y"], Y, what="Y")
    if ln_fp64:
        # fp64 statistics in the oracle's op order: only the row-sum order differs
        np.testing.assert_array_equal(g["y"], Y, err_msg="Y (ln_fp64) not bit-exact")
    # the production (non-debug) kernels give the same Y
    y2 = layer(xd, residual=rd)
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y2.cpu().numpy(), g["y"], err_msg="run != run_debug")
    if e2e:
        ref = oracle.mlp(L, X, R=R)
        _tier_int8(g["y"], ref, what="Y end-to-end")
    return flips


@pytest.mark.parametrize("C,T", [(96, 1000), (128, 300), (192, 257), (256, 129), (384, 200),
                                 (512, 131), (768, 257), (1024, 100), (1536, 129)])
def test_parity_relu_paper_mode(dev, C, T):
    """The paper's GELU-less block: ReLU, no FC1 bias, symmetric zero points."""
    _run_and_check(dev, _layer(C, 1000 + C), T)


@pytest.mark.parametrize("C,T", [(96, 1000), (256, 129), (384, 200), (768, 257), (1536, 129)])
def test_parity_relu_ln_fp64(dev, C, T):
    """ln_fp64 = 1: LayerNorm statistics and normalisation in fp64, the oracle's order (O5)."""
    _run_and_check(dev, _layer(C, 1000 + C), T, ln_fp64=True)


@pytest.mark.parametrize("C,T", [(96, 513), (384, 130), (768, 129)])
def test_parity_gelu_control(dev, C, T):
    """GELU control epilogue (the fused op the paper removes)."""
    _run_and_check(dev, _layer(C, 2000 + C, act=1, bias=True), T)


@pytest.mark.parametrize("C,T,zx,zh,zy", [(96, 300, -7, 0, 3), (192, 200, 0, -128, 0), (384, 150, 5, -7, -2)])
def test_parity_zero_points_and_bias(dev, C, T, zx, zh, zy):
    """Asymmetric activation zero points (reading R5) and an FC1 bias (north-star op #5)."""
    _run_and_check(dev, _layer(C, 3000 + C, bias=True, zx=zx, zh=zh, zy=zy), T)


@pytest.mark.parametrize("C,T", [(96, 200), (768, 131)])
def test_parity_fp32_residual(dev, C, T):
    """fp32 residual operand of op #6 (reading R3) and the residual_out tap."""
    _run_and_check(dev, _layer(C, 4000 + C), T, resid=True)


@pytest.mark.parametrize("T", [1, 2, 127, 128, 129, 255, 256])
def test_parity_tile_edges(dev, T):
    """Ragged token tails around the 128-row tile."""
    _run_and_check(dev, _layer(192, 5000), T)


@pytest.mark.parametrize("C,T,act,bias,zx,zh", [
    (96, 1000, 0, False, 0, 0), (192, 257, 1, True, 0, 0), (384, 200, 0, True, -7, 0),
    (768, 131, 1, False, 0, -128), (256, 129, 0, False, 5, -7), (1536, 129, 0, False, 0, 0)])
def test_parity_op5_unfused(dev, C, T, act, bias, zx, zh):
    """SURVEY.md §8(f) NEXT-1, the FasterTransformer layout: FC1
    writes A1 to HBM and op #5 runs as a separate kernel.  Same arithmetic: A1, Hq (ReLU), A2, z
    bit-exact; GELU Hq and Y within the tiers."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 6000 + C, act=act, bias=bias, zx=zx, zh=zh)
    _run_and_check(dev, L, T, op5_unfused=True)
    assert SwinMlpInt8Layer(L, device=0, op5_unfused=True).plan()["fused"] == 0


@pytest.mark.parametrize("C,T,bias,zh", [(96, 1000, False, 0), (384, 300, True, 0), (768, 129, False, -128),
                                         (1536, 77, False, 0)])
def test_parity_shift_gelu_control(dev, C, T, bias, zh):
    """SURVEY.md §8(f) NEXT-4's third control: I-ViT's integer shift-GELU (R28), which needs
    each token row's max before any output -- so it always runs unfused: FC1 -> A1 -> row-max op #5
    kernel -> FC2.  A1, Hq, A2, z bit-exact; Y within the op #6 tier."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer, lib
    L = _layer(C, 6200 + C, act=synth.ACT_SHIFT_GELU, bias=bias, zh=zh)
    _run_and_check(dev, L, T)
    assert lib().swin_mlp_int8_launches_per_run(SwinMlpInt8Layer(L, device=0).handle) == 3


def test_op5_unfused_matches_fused_plan(dev):
    """Same Y from the unfused (3-kernel) and the production plan on the same inputs (fp64 LN:
    the one-kernel and two-kernel plans order their fp32 row statistics differently)."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer, lib
    for C, T, act in ((96, 3000, 0), (384, 1000, 0), (192, 700, 1)):
        L = _layer(C, 6100 + C, act=act)
        x = torch.from_numpy(synth.make_activations(L, T, 9)).to(dev)
        a = SwinMlpInt8Layer(L, device=0, ln_fp64=True)
        b = SwinMlpInt8Layer(L, device=0, ln_fp64=True, op5_unfused=True)
        ya, yb = a(x), b(x)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(ya.cpu().numpy(), yb.cpu().numpy())
        assert lib().swin_mlp_int8_launches_per_run(b.handle) == 3


@pytest.mark.parametrize("C,T", [(384, 148 * 256 * 2 + 77), (512, 148 * 256 + 300), (448, 1000), (320, 129)])
def test_ln_pair_plan(dev, C, T, monkeypatch):
    """FC2 + op #6 on a CTA pair (opt-in SWIN_MLP_LN_PAIR: cta_group::2, M = 256, whole row in
    each CTA's TMEM, one accumulator buffer): several tiles per CTA (accumulator phase), odd
    m-tile counts."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    monkeypatch.setenv("SWIN_MLP_LN_PAIR", "1")
    L = _layer(C, 8800 + C)
    pl = SwinMlpInt8Layer(L, device=0).plan()
    assert pl["fused"] == 0 and pl["fc2_cs"] == 1 and pl["fc2_bn"] == C, pl
    _run_and_check(dev, L, T, e2e=False)
    _run_and_check(dev, _layer(C, 8900 + C, act=1, bias=True, zx=-3, zh=5, zy=2), min(T, 700), e2e=False,
                   resid=True)


def test_t_zero_is_noop(dev):
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    layer = SwinMlpInt8Layer(_layer(96, 1), device=0)
    x = torch.empty((0, 96), dtype=torch.int8, device=dev)
    y = layer(x)
    torch.cuda.synchronize()
    assert y.shape == (0, 96)


def test_folded_constants_match_oracle(dev):
    """O0 on the device side: the library's folded fp32 constants equal the oracle's bit for bit."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(384, 6000, zx=-3, zh=-128)
    layer = SwinMlpInt8Layer(L, device=0)
    m1, ih, m2, iy, w1, w2 = layer.constants()
    om1, oih, om2, oiy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
    np.testing.assert_array_equal(m1, om1)
    np.testing.assert_array_equal(m2, om2)
    assert np.float32(ih) == np.float32(oih) and np.float32(iy) == np.float32(oiy)
    np.testing.assert_array_equal(w1, L.w1.astype(np.int64).sum(1))
    np.testing.assert_array_equal(w2, L.w2.astype(np.int64).sum(1))


def test_shard_concat_equals_unsharded(dev, monkeypatch):
    """Tokens are independent rows: running shards separately and
    concatenating equals the unsharded run bit-exactly (the multi-GPU invariant) while the
    shards run the same launch plan.  The plan is a function of T (the few-tile plans for
    runs of at most a few m-tiles), so this arm pins the many-tile plans
    (SWIN_MLP_SMALL=0); the next test covers a plan switch."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    monkeypatch.setenv("SWIN_MLP_SMALL", "0")
    L = _layer(384, 7000)
    T = 1000
    X = torch.from_numpy(synth.make_activations(L, T, 9)).to(dev)
    layer = SwinMlpInt8Layer(L, device=0)
    full = layer(X).cpu()
    parts = [layer(X[a:b].contiguous()).cpu() for a, b in ((0, 384), (384, 513), (513, 1000))]
    torch.cuda.synchronize()
    assert torch.equal(full, torch.cat(parts))
    # row permutation equivariance
    perm = torch.randperm(T, generator=torch.Generator().manual_seed(1))
    yp = layer(X[perm.to(dev)].contiguous()).cpu()
    assert torch.equal(yp, full[perm])


@pytest.mark.parametrize("ln_fp64", [False, True])
def test_shard_concat_across_plan_switch(dev, ln_fp64):
    """Shards small enough for the few-tile plans (FC1 BN = 64 tiles, op #6 on an 8-CTA
    cluster) against the unsharded many-tile run: Hq is integer/elementwise work and the
    same bit for bit under any tiling; Y differs only in the LayerNorm statistics' fp32
    summation order (the row split across 8 instead of 2 CTAs), so it is within the Y tier
    (R15) with fp32 statistics and bit-exact with ln_fp64."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(384, 7001)
    T = 1000
    X = torch.from_numpy(synth.make_activations(L, T, 10)).to(dev)
    layer = SwinMlpInt8Layer(L, device=0, ln_fp64=ln_fp64)
    full = layer.run_debug(X)
    cuts = ((0, 49), (49, 177), (177, 1000))
    parts = [layer.run_debug(X[a:b].contiguous()) for a, b in cuts]
    torch.cuda.synchronize()
    hq = torch.cat([p["hidden"].cpu() for p in parts])
    assert torch.equal(full["hidden"].cpu(), hq)
    y = torch.cat([p["y"].cpu() for p in parts]).numpy()
    if ln_fp64:
        np.testing.assert_array_equal(full["y"].cpu().numpy(), y)
    else:
        _tier_int8(y, full["y"].cpu().numpy(), what="Y across plans")


@pytest.mark.parametrize("C,T,plan", [(384, 49, "few_tile"), (512, 49, "few_tile"), (768, 49, "few_tile"),
                                      (768, 128, "few_tile"), (768, 200, "few_tile"), (1024, 49, "few_tile"),
                                      (1536, 49, "default"), (384, 1, "few_tile"), (768, 17, "few_tile")])
def test_parity_few_tile_plans(dev, C, T, plan, monkeypatch):
    """The few-tile plans chosen per run for one or two m-tiles against the oracle, every output
    element (runs of <= 64 tokens take the one-launch plan unless SWIN_MLP_TINY=0).  The plan each
    case runs is asserted: at C = 1536 the default FC1 CTA-pair plan already spreads one m-tile
    over 48 CTAs (>= num_sms / 4), so that case is the default plan (with split-K op #6) at T = 49."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    monkeypatch.setenv("SWIN_MLP_TINY", "0")
    assert SwinMlpInt8Layer(_layer(C, 7100 + C + T), device=0).plan(T)["run_plan"] == plan
    _run_and_check(dev, _layer(C, 7100 + C + T), T, x_seed=T)
    _run_and_check(dev, _layer(C, 7200 + C + T, act=1, bias=True, zx=-5, zh=3, zy=2), T, x_seed=T + 1,
                   resid=True, e2e=False)


@pytest.mark.parametrize("C,T", [(384, 49), (512, 64), (768, 49), (768, 1), (768, 17), (1024, 33), (1536, 49),
                                 (640, 49)])
def test_parity_one_launch_plan(dev, C, T):
    """The one-launch plan for runs of <= 64 tokens (small_mlp.cuh; configs[0]: one 7x7 window,
    T = 49, C = 768): H/128 CTAs each own 128 hidden columns, FC2 partials summed exactly, op #6
    per row by one warp.  A1, Hq, A2, z bit-exact; Y within the tier; GELU, bias, zero points and
    the fp32 residual on the second case.  Back-to-back runs exercise the counter reset."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 7500 + C + T)
    assert SwinMlpInt8Layer(L, device=0).plan(T)["run_plan"] == "one_launch"
    for rep in range(2):
        _run_and_check(dev, L, T, x_seed=T + rep)
    _run_and_check(dev, _layer(C, 7600 + C + T, act=1, bias=True, zx=-5, zh=3, zy=2), T, x_seed=T + 1,
                   resid=True, e2e=False)


@pytest.mark.parametrize("C,T,q", [(768, 49, 4), (768, 64, 6), (768, 33, 8), (1024, 49, 8), (384, 17, 4)])
def test_one_launch_cluster_sizes(dev, C, T, q, monkeypatch):
    """The one-launch plan's cluster split at other cluster sizes (SWIN_MLP_TINY_Q: the smallest
    valid Q >= q): more peers per Hq exchange (DSMEM bulk copies into up to 7 peers), narrower
    column groups per CTA, fewer-way L2 sums.  A1, Hq, A2, z bit-exact, Y in tier."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    monkeypatch.setenv("SWIN_MLP_TINY_Q", str(q))
    L = _layer(C, 7700 + C + T + q)
    plan = SwinMlpInt8Layer(L, device=0).plan(T)
    assert plan["run_plan"] == "one_launch" and plan["fc2_cs"] >= q and C % plan["fc2_cs"] == 0
    _run_and_check(dev, L, T, x_seed=T + q, e2e=False)


def test_run_host_matches_device(dev):
    """The end-to-end host-buffer entry point (H2D, run, D2H inside the library)."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(192, 8000)
    T = 700
    Xn = synth.make_activations(L, T, 3)
    layer = SwinMlpInt8Layer(L, device=0)
    xh = torch.from_numpy(Xn).pin_memory()
    yh = torch.empty((T, 192), dtype=torch.int8).pin_memory()
    layer.run_host(xh, yh)
    torch.cuda.synchronize()
    yd = layer(xh.to(dev)).cpu()
    torch.cuda.synchronize()
    assert torch.equal(yh, yd)


def test_run_host_pipelined_and_batch(dev):
    """run_host over several token chunks (T > one chunk) and run_host_batch over layers of
    different widths (one pipeline over all their chunks) give the device-path outputs."""
    import paper_2402_01169_b200 as P
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    specs = [(_layer(96, 8100), 40000), (_layer(384, 8101), 5000), (_layer(768, 8102), 333)]
    layers, xs, ys, refs = [], [], [], []
    for L, T in specs:
        layer = SwinMlpInt8Layer(L, device=0)
        xh = torch.from_numpy(synth.make_activations(L, T, 4)).pin_memory()
        refs.append(layer(xh.to(dev)).cpu())
        layers.append(layer)
        xs.append(xh)
        ys.append(torch.zeros((T, L.C), dtype=torch.int8).pin_memory())
    torch.cuda.synchronize()
    # pipelined single-layer calls
    for layer, xh, yh, ref in zip(layers, xs, ys, refs):
        layer.run_host(xh, yh)
        torch.cuda.synchronize()
        assert torch.equal(yh, ref)
        yh.zero_()
    # one batch over all layers
    Ts = [x.shape[0] for x in xs]
    hs = [l.handle for l in layers]
    n = P.swin_mlp_int8_host_batch_workspace_bytes(hs, Ts)
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream(dev).cuda_stream
    P.swin_mlp_int8_run_host_batch(hs, xs, ys, Ts, ws.data_ptr(), n, s)
    torch.cuda.synchronize()
    for yh, ref in zip(ys, refs):
        assert torch.equal(yh, ref)


def test_full_size_config2_sampled(dev):
    """BASELINE configs[1] (Swin-T, four stage MLPs, batch 64) at full size, in the
    bench's launch configuration: sampled rows (first/last tile, tile boundaries,
    random) against the oracle computed row by row."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    rng = np.random.default_rng(11)
    for L, T, xs in synth.swin_t_batch64_layers():
        X = synth.make_activations(L, T, xs)
        layer = SwinMlpInt8Layer(L, device=0)
        y = layer(torch.from_numpy(X).to(dev)).cpu().numpy()
        torch.cuda.synchronize()
        rows = np.unique(np.concatenate([np.arange(0, 128), np.arange(T - 128, T),
                                         np.arange(127, T, 128)[:200], np.arange(128, T, 128)[:200],
                                         rng.integers(0, T, 1500)]))
        ref = oracle.mlp(L, X, rows=rows)
        _tier_int8(y[rows], ref, what=f"config2 C={L.C} sampled rows")


def test_multiple_handles_interleaved(dev):
    """Handles of different shapes coexist: create all first, then run in any order
    (regression: a per-kernel launch attribute set by one handle must not break another)."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    Ls = [_layer(C, 9000 + C) for C in (768, 96, 1536, 192)]
    layers = [SwinMlpInt8Layer(L, device=0) for L in Ls]
    for L, layer in list(zip(Ls, layers))[::-1]:
        X = synth.make_activations(L, 150, 4)
        y = layer(torch.from_numpy(X).to(dev)).cpu().numpy()
        torch.cuda.synchronize()
        _tier_int8(y, oracle.mlp(L, X), what=f"C={L.C}")


@pytest.mark.parametrize("C", [96, 256, 384])
def test_parity_extreme_accumulators(dev, C):
    """Saturated inputs drive |A1| to its bound (128*127*C: 4.16e6 at C=256, just under
    the 2^22 limit of the exact small-K int->float path) and saturate Hq and Y."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 9100 + C)
    rng = np.random.default_rng(C)
    L.w1 = np.where(rng.random(L.w1.shape) < 0.5, 127, -127).astype(np.int8)
    L.w1[: L.H // 2] = 127                       # half the hidden units see +127 everywhere
    L.w2 = np.where(rng.random(L.w2.shape) < 0.5, 127, -127).astype(np.int8)
    T = 300
    X = np.full((T, C), -128, np.int8)
    X[T // 2:] = 127
    # near-constant LayerNorm rows (|mean| >> std): exercises the corrected two-pass fp32 variance
    layer = SwinMlpInt8Layer(L, device=0)
    taps = layer.run_debug(torch.from_numpy(X).to(dev))
    torch.cuda.synchronize()
    a1 = oracle.gemm_i8(X, L.w1, L.z_x)
    assert np.abs(a1).max() >= 128 * 127 * C * 0.99
    np.testing.assert_array_equal(taps["acc1"].cpu().numpy(), a1)
    m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
    np.testing.assert_array_equal(taps["hidden"].cpu().numpy(), oracle.ep5(a1, m1, L.b1, ih, L.z_h))
    _tier_int8(taps["y"].cpu().numpy(), oracle.mlp(L, X), what="Y extreme")


@pytest.mark.parametrize("C,zx", [(512, 0), (768, 0), (768, -3)])
def test_parity_weight_bound_small_k(dev, C, zx):
    """The exact magic-number int->float path of op #5 is chosen from the weights' own bound
    (128 + |z_x|) * max_n sum_k |W1[n][k]| < 2^22.  Hidden unit 0 sits just under that bound and
    is driven to it (|A1| = 4194176 or the largest multiple the zero point allows); unit 1 is just
    over it for the bound-free path's sake on a second handle.  acc1 and Hq bit-exact."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 9300 + C, zx=zx)
    lim = (1 << 22) // (128 + abs(zx))            # row |sum| must stay below this
    row = np.zeros(C, np.int8)
    n127 = (lim - 1) // 127
    row[:n127] = 127
    row[n127] = (lim - 1) - 127 * n127            # sum |W1[0]| = lim - 1
    L.w1[0] = row
    L.w1[1] = -row
    T = 260
    X = synth.make_activations(L, T, 3)
    X[:130, :n127 + 1] = -128                    # drives A1[:, 0] to -(128 + z_x) * (lim - 1)
    X[130:, :n127 + 1] = 127
    for variant in (0, 1):
        if variant:
            L.w1[2] = 127                          # bound exceeded: the I2F path
        layer = SwinMlpInt8Layer(L, device=0)
        taps = layer.run_debug(torch.from_numpy(X).to(dev))
        torch.cuda.synchronize()
        a1 = oracle.gemm_i8(X, L.w1, L.z_x)
        if not variant:
            assert np.abs(a1).max() < (1 << 22) and np.abs(a1[:, 0]).max() >= (1 << 22) - 2 * 255 * 128
        np.testing.assert_array_equal(taps["acc1"].cpu().numpy(), a1)
        m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
        np.testing.assert_array_equal(taps["hidden"].cpu().numpy(), oracle.ep5(a1, m1, L.b1, ih, L.z_h))


# ---- one-kernel plan (fused_mlp.cuh, C <= 256) vs the two-kernel plan ---------------------------

@pytest.mark.parametrize("C,fused", [(96, 1), (128, 1), (192, 1), (256, 1), (384, 0), (512, 0), (768, 0)])
def test_plan_selection(dev, C, fused, monkeypatch):
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 7000 + C)
    assert SwinMlpInt8Layer(L, device=0).plan()["fused"] == fused
    monkeypatch.setenv("SWIN_MLP_NO_FUSED", "1")
    assert SwinMlpInt8Layer(L, device=0).plan()["fused"] == 0


@pytest.mark.parametrize("C,T", [(96, 1000), (192, 257), (256, 129), (384, 200)])
def test_two_kernel_plan_small_c(dev, C, T, monkeypatch):
    """The two-kernel plan stays correct for the channel counts the one-kernel plan now takes."""
    monkeypatch.setenv("SWIN_MLP_NO_FUSED", "1")
    _run_and_check(dev, _layer(C, 1000 + C), T)
    _run_and_check(dev, _layer(C, 3000 + C, bias=True, zx=-5, zh=-128, zy=2), T)


@pytest.mark.parametrize("C,T", [(96, 148 * 128 * 2 + 77), (192, 148 * 128 + 1000), (256, 148 * 128 + 129)])
def test_fused_persistent_multi_tile(dev, C, T):
    """Several m-tiles per CTA (X-slot reuse, TMEM / Hq buffer phases across tiles), resident and
    streamed weights, ragged tail."""
    _run_and_check(dev, _layer(C, 8000 + C), T, e2e=False)


@pytest.mark.parametrize("C,T", [(96, 3000), (192, 1000), (384, 300)])
def test_fused_gelu_and_ln_fp64(dev, C, T):
    _run_and_check(dev, _layer(C, 9000 + C, act=1, bias=True, zh=-3), T)
    _run_and_check(dev, _layer(C, 9100 + C), T, ln_fp64=True)


@pytest.mark.parametrize("C,T", [(768, 3 * 128 - 51), (512, 20 * 128 + 77)])
def test_fc1_cta_pair(dev, C, T):
    """FC1 on a CTA pair (cta_group::2, M = 256): odd m-tile counts (the last pair's second
    tile entirely out of range), several pair tiles per cluster, ReLU and GELU, zero points."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 9500 + C)
    assert SwinMlpInt8Layer(L, device=0).plan()["fc1_pair"] == 1
    _run_and_check(dev, L, T, e2e=False)
    _run_and_check(dev, _layer(C, 9600 + C, act=1, bias=True, zx=-5, zh=-3, zy=2), T, e2e=False)


@pytest.mark.parametrize("C,T,env", [
    (512, 9 * 128 + 1, {"SWIN_MLP_NO_YIN": "1", "SWIN_MLP_LN_PAIR": "0"}),   # op #6 separate Y staging
    (512, 9 * 128 + 1, {"SWIN_MLP_LN_CS": "4", "SWIN_MLP_LN_PAIR": "0"}),    # op #6 4-CTA column split
    (384, 98 * 128, {}),                                              # few tiles: the pair op #6 plan
    (384, 150 * 128 + 3, {}),                                         # more: the column-split plan
    (1024, 7 * 128 + 100, {}),                                        # op #6 yin at cs = 4, BN = 256
])
def test_gemm_plan_variants(dev, C, T, env, monkeypatch):
    """Two-kernel plan variants: op #6 with and without Y staged over its x
    tile, forced cluster sizes, the CTA-pair op #6 and the column-split plan;
    ReLU paper mode and GELU with bias and zero points, bit-exact / tiered against the oracle."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    L = _layer(C, 9700 + C)
    plan = SwinMlpInt8Layer(L, device=0).plan()
    assert plan["fused"] == 0
    if "SWIN_MLP_LN_CS" in env:
        assert plan["fc2_cs"] == int(env["SWIN_MLP_LN_CS"])
    _run_and_check(dev, L, T, e2e=False)
    _run_and_check(dev, _layer(C, 9800 + C, act=1, bias=True, zx=-5, zh=-3, zy=2), T, e2e=False)


# ---- NEXT-2: proj GEMM + fused op #4 (+ LN2) ---------------------------------------------------

@pytest.mark.parametrize("C,T,za,zy,bias,ln64", [
    (96, 3000, 0, 0, True, False), (128, 129, -3, 2, False, False), (192, 1000, 0, 0, True, True),
    (256, 257, 5, -1, True, False), (384, 1500, 0, 0, True, False), (512, 20 * 128 + 77, 0, 0, True, False),
    (768, 300, -7, 0, True, True), (1024, 7 * 128 + 100, 0, 0, True, False),
])
def test_parity_proj_op4(dev, C, T, za, zy, bias, ln64):
    """swin_proj_int8_* (Fig. 1 lines 63-70, reading R18) against oracle.proj_op4:
    A int32 and z (the fp32 residual stream handed to the MLP) bit-exact, yhat and Y in tier."""
    from paper_2402_01169_b200 import SwinProjInt8Layer
    P = synth.make_proj(C, 9900 + C, bias=bias, z_a=za, z_y=zy)
    A_in = synth.make_attn_out(P, T, 17)
    R = synth.make_residual(T, C, 18)
    layer = SwinProjInt8Layer(P, device=0, ln_fp64=ln64)
    zo = torch.empty((T, C), dtype=torch.float32, device=dev)
    taps = layer.run_debug(torch.from_numpy(A_in).to(dev), torch.from_numpy(R).to(dev), residual_out=zo)
    torch.cuda.synchronize()
    Y, yh, z, A = oracle.proj_op4(P, A_in, R)
    np.testing.assert_array_equal(taps["acc"].cpu().numpy(), A)
    np.testing.assert_array_equal(zo.cpu().numpy(), z)
    _tier_yhat(taps["ln_out"].cpu().numpy(), yh)
    _tier_int8(taps["y"].cpu().numpy(), Y, what=f"proj Y C={C}")
    y2 = layer(torch.from_numpy(A_in).to(dev), torch.from_numpy(R).to(dev))   # plain run == debug run
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y2.cpu().numpy(), taps["y"].cpu().numpy())


def test_proj_op4_feeds_mlp(dev):
    """One Swin MLP half-block end to end on the GPU: proj + op #4 (+LN2) -> MLP with the fp32
    residual stream z, against the oracle composition (bit-exact z chain, Y in tier)."""
    from paper_2402_01169_b200 import SwinProjInt8Layer, SwinMlpInt8Layer
    C, T = 384, 700
    P = synth.make_proj(C, 9950)
    L = synth.make_layer(C, 9951)
    L.s_x = P.s_y          # the MLP consumes op #4's quantized LN2 output
    A_in = synth.make_attn_out(P, T, 19)
    R = synth.make_residual(T, C, 20)
    proj, mlp = SwinProjInt8Layer(P, device=0), SwinMlpInt8Layer(L, device=0)
    z1 = torch.empty((T, C), dtype=torch.float32, device=dev)
    x = proj(torch.from_numpy(A_in).to(dev), torch.from_numpy(R).to(dev), residual_out=z1)
    z2 = torch.empty((T, C), dtype=torch.float32, device=dev)
    y = mlp(x, residual=z1, residual_out=z2)
    torch.cuda.synchronize()
    Yp, _, zp, _ = oracle.proj_op4(P, A_in, R)
    _tier_int8(x.cpu().numpy(), Yp, what="op #4 Y")
    xin = x.cpu().numpy()                          # the MLP oracle on the GPU's own int8 input
    np.testing.assert_array_equal(z1.cpu().numpy(), zp)
    _tier_int8(y.cpu().numpy(), oracle.mlp(L, xin, R=zp), what="MLP Y")


def test_proj_requires_residual(dev):
    from paper_2402_01169_b200 import SwinProjInt8Layer, SwinMlpError
    P = synth.make_proj(96, 9960)
    layer = SwinProjInt8Layer(P, device=0)
    a = torch.zeros((10, 96), dtype=torch.int8, device=dev)
    with pytest.raises(SwinMlpError):
        layer(a, None)


def test_plan_for_reports_the_run_plan(dev):
    """swin_mlp_int8_plan_for: a one-window run (T = 49) at C = 768 takes the few-tile plans
    (FC1 BN = 64 single-CTA tiles, op #6 on an 8-CTA cluster), a full-stage run the defaults."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    layer = SwinMlpInt8Layer(_layer(768, 7300), device=0)
    window, small, big = layer.plan(49), layer.plan(100), layer.plan(200704)
    assert window["run_plan"] == "one_launch" and window["fc1_bn"] == 3072 // 128   # CTAs
    assert small["run_plan"] == "few_tile" and small["fc1_bn"] == 64 and small["fc1_pair"] == 0
    assert small["fc2_cs"] == 8 and small["fc2_bn"] == 96
    assert big["run_plan"] == "default"
    assert big["fc2_ksplit"] == 1 and small["fc2_ksplit"] > 1   # split-K: one m-tile only
    assert {k: v for k, v in big.items() if k not in ("run_plan", "fc2_ksplit")} == layer.plan()


# ---- round-to-nearest-even ties forced through the GPU (reading R2) --------------------------

def _tie_layer(C, seed, zh=0, zy=0):
    """Power-of-two scales so every fp32 op of both epilogues is exact and RNE ties occur in
    bulk (tests/golden/ep5_pow2_table.txt's scales): s_x = 2^-4, s_w1 = 2^-6 -> m1 = 2^-10,
    s_h = 2^-7 -> inv_h = 128, so v = A1 / 8 (no FC1 bias) and every A1 = 4 (mod 8) is an exact
    .5 tie of op #5's Q.  Op #6: s_y = 2^-4 (inv_y = 16); gamma = 0 on the even columns makes
    yhat == beta exactly there, and beta = (k + 1/2) / 16 puts Y's Q on a tie for every such
    element (k spans the clamp range too); odd columns keep a real LayerNorm."""
    rng = np.random.default_rng(seed)
    L = synth.make_layer(C, seed, z_h=zh, z_y=zy)
    H = L.H
    L.s_x = 2.0 ** -4
    L.w1 = rng.integers(-1, 2, (H, C)).astype(np.int8)
    L.s_w1 = np.full(H, 2.0 ** -6, np.float32)
    L.s_h = 2.0 ** -7
    L.w2 = rng.integers(-20, 21, (C, H)).astype(np.int8)
    L.s_w2 = np.full(C, 2.0 ** -6, np.float32)
    L.s_y = 2.0 ** -4
    L.gamma = np.where(np.arange(C) % 2 == 0, 0.0, L.gamma).astype(np.float32)
    k = rng.integers(-140, 140, C)
    L.beta = np.where(np.arange(C) % 2 == 0, (k + 0.5) / 16.0, L.beta).astype(np.float32)
    return L


@pytest.mark.parametrize("C,T,zh,zy", [(96, 1000, 0, 0), (192, 300, -128, 3), (384, 700, 0, -2),
                                       (768, 49, 0, 0), (768, 1000, -7, 0), (1536, 129, 0, 1)])
def test_parity_rne_ties(dev, C, T, zh, zy):
    """Exact .5 ties through both epilogues on the GPU, every plan family (one-kernel C <= 256,
    two-kernel, few-tile T = 49): Hq bit-exact against the oracle (whose Q is pinned by the
    golden tie tables), and Y bit-exact on the tie columns; a half-away-from-zero rounding
    anywhere would fail."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _tie_layer(C, 9400 + C, zh=zh, zy=zy)
    rng = np.random.default_rng(C + T)
    X = rng.integers(-8, 9, (T, C)).astype(np.int8)
    layer = SwinMlpInt8Layer(L, device=0)
    taps = layer.run_debug(torch.from_numpy(X).to(dev))
    torch.cuda.synchronize()
    a1 = oracle.gemm_i8(X, L.w1, L.z_x)
    ties5 = int((((a1 % 8) == 4) & (a1 > 0)).sum())
    assert ties5 > 0.02 * a1.size, ties5           # plenty of positive (un-ReLU'd) ties
    np.testing.assert_array_equal(taps["acc1"].cpu().numpy(), a1)
    m1, ih, m2, iy = oracle.fold_constants(L.s_x, L.s_w1, L.s_h, L.s_w2, L.s_y)
    assert ih == 128.0 and iy == 16.0
    hq = taps["hidden"].cpu().numpy()
    np.testing.assert_array_equal(hq, oracle.ep5(a1, m1, L.b1, ih, L.z_h), err_msg="Hq at ties")
    Y, _, _ = oracle.ep6(taps["acc2"].cpu().numpy(), m2, L.b2, X, L.s_x, L.z_x, L.gamma, L.beta, L.eps, iy, L.z_y)
    y = taps["y"].cpu().numpy()
    np.testing.assert_array_equal(y[:, ::2], Y[:, ::2], err_msg="Y at ties (gamma = 0 columns)")
    want = np.clip(np.rint(L.beta.astype(np.float64) * 16) + zy, -128, 127)[::2]
    np.testing.assert_array_equal(Y[0, ::2], want.astype(np.int8))   # the oracle rounds the ties to even
    _tier_int8(y, Y, what="Y")
    y2 = layer(torch.from_numpy(X).to(dev))
    torch.cuda.synchronize()
    np.testing.assert_array_equal(y2.cpu().numpy(), y, err_msg="run != run_debug")


# ---- full-size sampled rows at the north-star and Swin-L stage shapes ----------------------------

@pytest.mark.parametrize("C,T", [(512, 25088), (1024, 6272), (128, 401408), (1536, 28800), (768, 72000)])
def test_full_size_stage_shapes_sampled(dev, C, T):
    """The Swin-B b128-per-GPU stage shapes (the north-star stack: C = 512 at T = 25088 runs the
    default op #6 plan -- CS = 2, BN = 256, Y staged over x -- for 18 of its 24 layers; C = 1024
    at 6272; C = 128 at 401408) and Swin-L 384^2 (C = 1536 at T = 28800 = b32 x 30 x 30; C = 768
    at 72000), in the bench's launch configuration, against the oracle on sampled rows (every
    tile boundary, first / last tile, random rows)."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 9990 + C)
    X = synth.make_activations(L, T, 33)
    layer = SwinMlpInt8Layer(L, device=0)
    if C == 512:
        pl = layer.plan(T)
        assert pl["run_plan"] == "default" and pl["fc2_cs"] == 2 and pl["fc2_bn"] == 256, pl
    y = layer(torch.from_numpy(X).to(dev)).cpu().numpy()
    torch.cuda.synchronize()
    rng = np.random.default_rng(C)
    rows = np.unique(np.concatenate([np.arange(0, 128), np.arange(T - 128, T), np.arange(127, T, 128)[:300],
                                     np.arange(128, T, 128)[:300], rng.integers(0, T, 1200)]))
    _tier_int8(y[rows], oracle.mlp(L, X, rows=rows), what=f"C={C} T={T} sampled rows")


def test_run_host_ragged_tail_is_chunking_invariant(dev):
    """run_host chunks at 4096 rows; a C = 768, T = 4145 call has a 49-row tail that
    alone would take the few-tile plan.  Every chunk is planned for the whole call's T, so the
    host path equals the device run bit for bit."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(768, 8200)
    T = 4096 + 49
    xh = torch.from_numpy(synth.make_activations(L, T, 4)).pin_memory()
    layer = SwinMlpInt8Layer(L, device=0)
    yd = layer(xh.to(dev)).cpu()
    yh = torch.empty((T, 768), dtype=torch.int8).pin_memory()
    layer.run_host(xh, yh)
    torch.cuda.synchronize()
    assert torch.equal(yh, yd)


def test_run_host_after_run_host_batch(dev):
    """run_host_batch (one small layer: few events) then run_host on the same handle."""
    import paper_2402_01169_b200 as P
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(384, 8300)
    layer = SwinMlpInt8Layer(L, device=0)
    T = 300
    xh = torch.from_numpy(synth.make_activations(L, T, 5)).pin_memory()
    ref = layer(xh.to(dev)).cpu()
    yb = torch.zeros((T, 384), dtype=torch.int8).pin_memory()
    n = P.swin_mlp_int8_host_batch_workspace_bytes([layer.handle], [T])
    ws = torch.empty(n, dtype=torch.uint8, device=dev)
    P.swin_mlp_int8_run_host_batch([layer.handle], [xh], [yb], [T], ws.data_ptr(), n,
                                   torch.cuda.current_stream(dev).cuda_stream)
    torch.cuda.synchronize()
    assert torch.equal(yb, ref)
    T2 = 40000
    xh2 = torch.from_numpy(synth.make_activations(L, T2, 6)).pin_memory()
    yh2 = torch.empty((T2, 384), dtype=torch.int8).pin_memory()
    layer.run_host(xh2, yh2)
    torch.cuda.synchronize()
    assert torch.equal(yh2, layer(xh2.to(dev)).cpu())


@pytest.mark.parametrize("C", [384, 512, 768])
def test_plan_hint_shard_concat_bit_exact(dev, C):
    """Multi-GPU invariant under any plan switch: with the plan hint set to the
    global T, fixed-batch token shards (8 GPUs' worth, the small per-GPU T that switches plans)
    concatenate to the unsharded run bit for bit, fp32 LayerNorm statistics included."""
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    L = _layer(C, 8400 + C)
    T = 8 * 196
    X = torch.from_numpy(synth.make_activations(L, T, 7)).to(dev)
    layer = SwinMlpInt8Layer(L, device=0)
    full = layer(X).cpu()
    layer.set_plan_hint(T)
    parts = [layer(X[r * 196:(r + 1) * 196].contiguous()).cpu() for r in range(8)]
    layer.set_plan_hint(0)
    torch.cuda.synchronize()
    assert torch.equal(full, torch.cat(parts))
