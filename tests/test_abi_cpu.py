"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/swin_mlp_int8.h declares, and rejects invalid descriptions
synchronously with SWIN_MLP_EINVAL and a last_error message (validation runs
before any CUDA call, SURVEY §8(b) "Errors")."""
import ctypes
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def P():
    import paper_2402_01169_b200 as P
    from paper_2402_01169_b200 import build
    build.build()
    P.lib()
    return P


def _declared():
    names = set()
    for h in sorted(os.listdir(os.path.join(ROOT, "include"))):
        if h.endswith(".h"):
            src = open(os.path.join(ROOT, "include", h)).read()
            src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
            names |= set(re.findall(r"\b(swin_(?:mlp|proj|op1|attn)_int8_[a-z_]+)\s*\(", src))
    return sorted(names)


def test_exports_every_declared_symbol(P):
    names = _declared()
    assert len(names) >= 10
    assert sorted(P.EXPORTS) == names
    L = P.lib()
    for n in names:
        assert hasattr(L, n), n


def test_sm100a_code_only():
    """The shipped kernels are sm_100a SASS with tcgen05 (UTCIMMA) and TMA (UTMALDG)."""
    import shutil
    import subprocess
    from paper_2402_01169_b200 import build
    lib = build.build()
    if not shutil.which("cuobjdump"):
        pytest.skip("no cuobjdump")
    out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "UTCIMMA" in out and "UTMALDG" in out and "LDTM" in out
    # every kernel instantiation carries the tcgen05 main loop (none folded to EXIT)
    funcs = out.split("Function : ")[1:]
    assert len(funcs) >= 16
    for f in funcs:
        name = f.split()[0]
        if "op5_unfused_kernel" in name or "op5_shiftgelu_kernel" in name:   # separate op #5 (NEXT-1/4)
            assert "LDG" in f and "STG" in f and "F2I" in f, name
        elif "op1_kernel" in name:         # op #1: HBM-bound LayerNorm + gather + Q (NEXT-4)
            assert "LDG" in f and "STG" in f and "SHFL" in f, name
        elif "attn_core_kernel" in name:   # op #3 core: warp mma.sync (IMMA) on 49 / 144-token windows
            assert "IMMA" in f and "MUFU.EX2" in f and "LDS" in f, name
        elif "small_mlp_kernel" in name:   # one-launch plan: FC2 partials by bulk reduce-add, op #6 by STG
            assert "UTCIMMA" in f and "LDTM" in f and "UTMALDG" in f and "UBLKRED" in f, name
        elif "mlp_gemm_kernelILi3E" in name:   # EP_ACC: FC1 storing int32 A1 from registers
            assert "UTCIMMA" in f and "LDTM" in f and "STG" in f, name
        else:
            assert "UTCIMMA" in f and "LDTM" in f and "UTMASTG" in f, name


def _desc(P, **kw):
    d = P.swin_mlp_int8_desc_t()
    C = kw.get("C", 96)
    H = kw.get("H", 4 * C)
    keep = []

    def arr(a):
        keep.append(a)
        return a.ctypes.data_as(ctypes.c_void_p).value

    d.C, d.H, d.act = C, H, kw.get("act", 0)
    d.x_scale, d.x_zero_point = kw.get("x_scale", 0.05), kw.get("x_zero_point", 0)
    d.w1 = arr(np.ones((H, C), np.int8)); d.w1_scale = arr(np.full(H, 0.01, np.float32))
    d.h_scale, d.h_zero_point = kw.get("h_scale", 0.02), kw.get("h_zero_point", 0)
    d.w2 = arr(np.ones((C, H), np.int8)); d.w2_scale = arr(np.full(C, 0.01, np.float32))
    d.ln_gamma = arr(np.ones(C, np.float32)); d.ln_beta = arr(np.zeros(C, np.float32))
    d.ln_eps = kw.get("ln_eps", 1e-5)
    d.y_scale, d.y_zero_point = kw.get("y_scale", 0.04), kw.get("y_zero_point", 0)
    d.device = 0
    if kw.get("null_w1"):
        d.w1 = None
    return d, keep


@pytest.mark.parametrize("kw,frag", [
    (dict(C=100), "multiple of 32"), (dict(C=96, H=80), "H="), (dict(act=7), "activation"),
    (dict(x_scale=0.0), "scales"), (dict(y_scale=float("inf")), "scales"), (dict(h_scale=1e-42), "scales"),
    (dict(ln_eps=0.0), "ln_eps"), (dict(x_zero_point=200), "zero point"), (dict(null_w1=True), "required"),
])
def test_create_rejects_invalid(P, kw, frag):
    d, keep = _desc(P, **kw)
    h = ctypes.c_void_p()
    st = P.lib().swin_mlp_int8_create(ctypes.byref(d), ctypes.byref(h))
    assert st == P.SWIN_MLP_EINVAL
    assert frag in P.last_error()
    assert h.value is None


def test_unsupported_size(P):
    d, keep = _desc(P, C=2048)
    h = ctypes.c_void_p()
    assert P.lib().swin_mlp_int8_create(ctypes.byref(d), ctypes.byref(h)) == P.SWIN_MLP_EUNSUPPORTED


def test_null_handle_paths(P):
    L = P.lib()
    assert L.swin_mlp_int8_run(None, None, None, None, None, 10, None, 0, None) == P.SWIN_MLP_EINVAL
    assert "NULL handle" in P.last_error()
    assert L.swin_mlp_int8_workspace_bytes(None, 10) == 0
    assert L.swin_mlp_int8_destroy(None) == P.SWIN_MLP_OK
    assert L.swin_mlp_int8_launches_per_run(None) == 0
    out = (ctypes.c_int32 * 20)()
    assert L.swin_mlp_int8_plan_for(None, 49, out) == -1


def _proj_desc(P, **kw):
    d = P.swin_proj_int8_desc_t()
    C = kw.get("C", 96)
    keep = []

    def arr(a):
        keep.append(a)
        return a.ctypes.data_as(ctypes.c_void_p).value

    d.C = C
    d.a_scale, d.a_zero_point = kw.get("a_scale", 0.035), kw.get("a_zero_point", 0)
    d.w = None if kw.get("null_w") else arr(np.ones((C, C), np.int8))
    d.w_scale = arr(np.full(C, 0.01, np.float32))
    d.b = None
    d.ln_gamma = arr(np.ones(C, np.float32)); d.ln_beta = arr(np.zeros(C, np.float32))
    d.ln_eps = kw.get("ln_eps", 1e-5)
    d.y_scale, d.y_zero_point = kw.get("y_scale", 0.04), kw.get("y_zero_point", 0)
    d.device = 0
    return d, keep


@pytest.mark.parametrize("kw,frag", [
    (dict(C=100), "multiple of 32"), (dict(a_scale=0.0), "scales"), (dict(y_scale=float("nan")), "scales"),
    (dict(ln_eps=-1.0), "ln_eps"), (dict(a_zero_point=-129), "zero point"), (dict(null_w=True), "required"),
])
def test_proj_create_rejects_invalid(P, kw, frag):
    """swin_proj_int8_create validates before touching the device (NEXT-2 entry points)."""
    d, keep = _proj_desc(P, **kw)
    h = ctypes.c_void_p()
    assert P.lib().swin_proj_int8_create(ctypes.byref(d), ctypes.byref(h)) == P.SWIN_MLP_EINVAL
    assert frag in P.last_error()
    assert h.value is None
    d, keep = _proj_desc(P, C=2048)
    assert P.lib().swin_proj_int8_create(ctypes.byref(d), ctypes.byref(h)) == P.SWIN_MLP_EUNSUPPORTED


def test_proj_null_handle_paths(P):
    L = P.lib()
    assert L.swin_proj_int8_run(None, None, None, None, None, 10, None) == P.SWIN_MLP_EINVAL
    assert "NULL handle" in P.last_error()
    assert L.swin_proj_int8_plan(None, None) == -1
    assert L.swin_proj_int8_destroy(None) == P.SWIN_MLP_OK


def test_no_cpu_fallback_in_product_path():
    """The product package never imports the oracle (or numpy-based math) — a CPU
    fallback would void every parity claim."""
    pkg = os.path.join(ROOT, "paper_2402_01169_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                s = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in s and "from oracle" not in s and "oracle_mlp" not in s, f


def test_attn_null_handle_paths(P):
    """NEXT-3 / NEXT-4 entry points: NULL handles and invalid descriptions fail before any launch."""
    L = P.lib()
    assert L.swin_op1_int8_run(None, None, 1, None, None) == P.SWIN_MLP_EINVAL
    assert "NULL handle" in P.last_error()
    assert L.swin_op1_int8_destroy(None) == P.SWIN_MLP_OK
    assert L.swin_attn_int8_run(None, None, 1, None, None, 0, None) == P.SWIN_MLP_EINVAL
    assert L.swin_attn_int8_workspace_bytes(None, 4) == 0
    assert L.swin_attn_int8_get_constants(None, None, None) == P.SWIN_MLP_EINVAL
    assert L.swin_attn_int8_destroy(None) == P.SWIN_MLP_OK
    d = P.swin_op1_int8_desc_t()
    d.C, d.M, d.shift, d.Hs, d.Ws, d.ln_eps, d.y_scale = 96, 7, 7, 14, 14, 1e-5, 0.04
    h = ctypes.c_void_p()
    assert L.swin_op1_int8_create(ctypes.byref(d), ctypes.byref(h)) == P.SWIN_MLP_EINVAL
    assert "shift" in P.last_error()
    a = P.swin_attn_int8_desc_t()
    a.C, a.heads, a.M, a.Hs, a.Ws = 96, 2, 7, 14, 14
    assert L.swin_attn_int8_create(ctypes.byref(a), ctypes.byref(h)) == P.SWIN_MLP_EINVAL
    assert "heads" in P.last_error()
