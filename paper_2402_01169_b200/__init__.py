"""paper_2402_01169_b200 — B200-native (sm_100a) fully-integer Swin MLP sub-layer
of arXiv 2402.01169 ("GELU-less quantized SWIN").

A thin ctypes binding over the C ABI in include/swin_mlp_int8.h (same names,
argument marshalling only).  Every step of the layer — FC1 GEMM, fused op #5
(ReLU or the GELU control), FC2 GEMM, fused op #6 (bias, residual, LayerNorm,
requantize) — runs in the CUDA kernels of libswin_mlp_int8.so.  There is no
CPU fallback: if the library is missing or was built for another target the
import of `lib()` raises.

PyTorch is used only for device memory and streams (see SwinMlpInt8Layer).
"""
import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SWIN_MLP_LIB") or os.path.join(HERE, "libswin_mlp_int8.so")

SWIN_MLP_OK = 0
SWIN_MLP_EINVAL = 1
SWIN_MLP_EUNSUPPORTED = 2
SWIN_MLP_ENOMEM = 3
SWIN_MLP_ECUDA = 4
SWIN_MLP_ACT_RELU = 0
SWIN_MLP_ACT_GELU_ERF = 1

# every symbol include/swin_mlp_int8.h declares
EXPORTS = [
    "swin_mlp_int8_create", "swin_mlp_int8_workspace_bytes", "swin_mlp_int8_run",
    "swin_mlp_int8_run_debug", "swin_mlp_int8_host_workspace_bytes", "swin_mlp_int8_run_host",
    "swin_mlp_int8_get_constants", "swin_mlp_int8_launches_per_run", "swin_mlp_int8_plan",
    "swin_mlp_int8_plan_for", "swin_mlp_int8_set_plan_hint",
    "swin_mlp_int8_profile_begin", "swin_mlp_int8_profile_end", "swin_mlp_int8_set_trace",
    "swin_mlp_int8_destroy", "swin_mlp_int8_last_error",
    "swin_mlp_int8_host_batch_workspace_bytes", "swin_mlp_int8_run_host_batch",
    "swin_op1_int8_create", "swin_op1_int8_run", "swin_op1_int8_destroy",
    "swin_attn_int8_create", "swin_attn_int8_workspace_bytes", "swin_attn_int8_run", "swin_attn_int8_run_debug",
    "swin_attn_int8_get_constants", "swin_attn_int8_profile_begin", "swin_attn_int8_profile_end",
    "swin_attn_int8_destroy",
    "swin_proj_int8_create", "swin_proj_int8_run", "swin_proj_int8_run_debug", "swin_proj_int8_plan",
    "swin_proj_int8_destroy",
]


class swin_mlp_int8_desc_t(ctypes.Structure):
    _fields_ = [
        ("C", ctypes.c_int32), ("H", ctypes.c_int32), ("act", ctypes.c_int32),
        ("x_scale", ctypes.c_float), ("x_zero_point", ctypes.c_int32),
        ("w1", ctypes.c_void_p), ("w1_scale", ctypes.c_void_p), ("b1", ctypes.c_void_p),
        ("h_scale", ctypes.c_float), ("h_zero_point", ctypes.c_int32),
        ("w2", ctypes.c_void_p), ("w2_scale", ctypes.c_void_p), ("b2", ctypes.c_void_p),
        ("ln_gamma", ctypes.c_void_p), ("ln_beta", ctypes.c_void_p), ("ln_eps", ctypes.c_float),
        ("y_scale", ctypes.c_float), ("y_zero_point", ctypes.c_int32),
        ("device", ctypes.c_int32), ("ln_fp64", ctypes.c_int32),
        ("op5_unfused", ctypes.c_int32), ("gelu_in_scale", ctypes.c_float),
    ]


class swin_proj_int8_desc_t(ctypes.Structure):
    _fields_ = [
        ("C", ctypes.c_int32), ("a_scale", ctypes.c_float), ("a_zero_point", ctypes.c_int32),
        ("w", ctypes.c_void_p), ("w_scale", ctypes.c_void_p), ("b", ctypes.c_void_p),
        ("ln_gamma", ctypes.c_void_p), ("ln_beta", ctypes.c_void_p), ("ln_eps", ctypes.c_float),
        ("y_scale", ctypes.c_float), ("y_zero_point", ctypes.c_int32),
        ("device", ctypes.c_int32), ("ln_fp64", ctypes.c_int32),
    ]


class swin_op1_int8_desc_t(ctypes.Structure):
    """include/swin_attn_int8.h (fused op #1, NEXT-4)."""
    _fields_ = [
        ("C", ctypes.c_int32), ("M", ctypes.c_int32), ("shift", ctypes.c_int32),
        ("Hs", ctypes.c_int32), ("Ws", ctypes.c_int32),
        ("ln_gamma", ctypes.c_void_p), ("ln_beta", ctypes.c_void_p), ("ln_eps", ctypes.c_float),
        ("y_scale", ctypes.c_float), ("y_zero_point", ctypes.c_int32), ("device", ctypes.c_int32),
    ]


class swin_attn_int8_desc_t(ctypes.Structure):
    """include/swin_attn_int8.h (QKV GEMM + op #2 -> Q.K + op #3 -> V.att, NEXT-3)."""
    _fields_ = [
        ("C", ctypes.c_int32), ("heads", ctypes.c_int32), ("M", ctypes.c_int32), ("shift", ctypes.c_int32),
        ("Hs", ctypes.c_int32), ("Ws", ctypes.c_int32),
        ("x_scale", ctypes.c_float), ("x_zero_point", ctypes.c_int32),
        ("w_qkv", ctypes.c_void_p), ("w_qkv_scale", ctypes.c_void_p), ("b_qkv", ctypes.c_void_p),
        ("q_scale", ctypes.c_float), ("k_scale", ctypes.c_float), ("v_scale", ctypes.c_float),
        ("rel_bias_table", ctypes.c_void_p),
        ("a_scale", ctypes.c_float), ("a_zero_point", ctypes.c_int32), ("device", ctypes.c_int32),
    ]


class SwinMlpError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"swin_mlp_int8 status {status}: {msg}")
        self.status = status


_lib = None


def lib():
    """Load the CUDA library (fails loudly if it is missing: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} not built; run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(LIB_PATH)
    P, i32, i64, sz = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_size_t
    L.swin_mlp_int8_create.argtypes = [ctypes.POINTER(swin_mlp_int8_desc_t), ctypes.POINTER(P)]
    L.swin_mlp_int8_create.restype = i32
    L.swin_mlp_int8_workspace_bytes.argtypes = [P, i64]
    L.swin_mlp_int8_workspace_bytes.restype = sz
    L.swin_mlp_int8_run.argtypes = [P, P, P, P, P, i64, P, sz, P]
    L.swin_mlp_int8_run.restype = i32
    L.swin_mlp_int8_run_debug.argtypes = [P, P, P, P, P, i64, P, sz, P, P, P, P, P]
    L.swin_mlp_int8_run_debug.restype = i32
    L.swin_mlp_int8_host_workspace_bytes.argtypes = [P, i64, i32]
    L.swin_mlp_int8_host_workspace_bytes.restype = sz
    L.swin_mlp_int8_run_host.argtypes = [P, P, P, P, i64, P, sz, P]
    L.swin_mlp_int8_run_host.restype = i32
    L.swin_mlp_int8_get_constants.argtypes = [P, P, P, P, P, P, P]
    L.swin_mlp_int8_get_constants.restype = i32
    L.swin_mlp_int8_launches_per_run.argtypes = [P]
    L.swin_mlp_int8_launches_per_run.restype = i32
    L.swin_mlp_int8_plan.argtypes = [P, P]
    L.swin_mlp_int8_plan.restype = i32
    L.swin_mlp_int8_plan_for.argtypes = [P, ctypes.c_int64, P]
    L.swin_mlp_int8_plan_for.restype = i32
    L.swin_mlp_int8_set_plan_hint.argtypes = [P, ctypes.c_int64]
    L.swin_mlp_int8_set_plan_hint.restype = i32
    L.swin_mlp_int8_profile_begin.argtypes = [P, i32]
    L.swin_mlp_int8_profile_begin.restype = i32
    L.swin_mlp_int8_profile_end.argtypes = [P, P, P, P]
    L.swin_mlp_int8_profile_end.restype = i32
    L.swin_mlp_int8_set_trace.argtypes = [P, P, i32]
    L.swin_mlp_int8_set_trace.restype = i32
    L.swin_mlp_int8_destroy.argtypes = [P]
    L.swin_mlp_int8_destroy.restype = i32
    L.swin_mlp_int8_host_batch_workspace_bytes.argtypes = [i32, P, P]
    L.swin_mlp_int8_host_batch_workspace_bytes.restype = sz
    L.swin_mlp_int8_run_host_batch.argtypes = [i32, P, P, P, P, P, sz, P]
    L.swin_mlp_int8_run_host_batch.restype = i32
    L.swin_proj_int8_create.argtypes = [ctypes.POINTER(swin_proj_int8_desc_t), ctypes.POINTER(P)]
    L.swin_proj_int8_create.restype = i32
    L.swin_proj_int8_run.argtypes = [P, P, P, P, P, i64, P]
    L.swin_proj_int8_run.restype = i32
    L.swin_proj_int8_run_debug.argtypes = [P, P, P, P, P, i64, P, P, P]
    L.swin_proj_int8_run_debug.restype = i32
    L.swin_proj_int8_plan.argtypes = [P, P]
    L.swin_proj_int8_plan.restype = i32
    L.swin_proj_int8_destroy.argtypes = [P]
    L.swin_proj_int8_destroy.restype = i32
    L.swin_op1_int8_create.argtypes = [ctypes.POINTER(swin_op1_int8_desc_t), ctypes.POINTER(P)]
    L.swin_op1_int8_create.restype = i32
    L.swin_op1_int8_run.argtypes = [P, P, i64, P, P]
    L.swin_op1_int8_run.restype = i32
    L.swin_op1_int8_destroy.argtypes = [P]
    L.swin_op1_int8_destroy.restype = i32
    L.swin_attn_int8_create.argtypes = [ctypes.POINTER(swin_attn_int8_desc_t), ctypes.POINTER(P)]
    L.swin_attn_int8_create.restype = i32
    L.swin_attn_int8_workspace_bytes.argtypes = [P, i64]
    L.swin_attn_int8_workspace_bytes.restype = sz
    L.swin_attn_int8_run.argtypes = [P, P, i64, P, P, sz, P]
    L.swin_attn_int8_run.restype = i32
    L.swin_attn_int8_run_debug.argtypes = [P, P, i64, P, P, sz, P, P, P, P]
    L.swin_attn_int8_run_debug.restype = i32
    L.swin_attn_int8_get_constants.argtypes = [P, P, P]
    L.swin_attn_int8_get_constants.restype = i32
    L.swin_attn_int8_profile_begin.argtypes = [P, i32]
    L.swin_attn_int8_profile_begin.restype = i32
    L.swin_attn_int8_profile_end.argtypes = [P, P, P, P]
    L.swin_attn_int8_profile_end.restype = i32
    L.swin_attn_int8_destroy.argtypes = [P]
    L.swin_attn_int8_destroy.restype = i32
    L.swin_mlp_int8_last_error.argtypes = []
    L.swin_mlp_int8_last_error.restype = ctypes.c_char_p
    _lib = L
    return L


def last_error() -> str:
    return lib().swin_mlp_int8_last_error().decode()


def _check(st):
    if st != SWIN_MLP_OK:
        raise SwinMlpError(st, last_error())


# ---- same-name thin wrappers over the C ABI (raw pointers as ints) -------------
def swin_mlp_int8_create(desc: swin_mlp_int8_desc_t) -> int:
    h = ctypes.c_void_p()
    _check(lib().swin_mlp_int8_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def swin_mlp_int8_workspace_bytes(h, T) -> int:
    return int(lib().swin_mlp_int8_workspace_bytes(h, T))


def swin_mlp_int8_run(h, x, residual, y, residual_out, T, workspace, workspace_bytes, stream):
    _check(lib().swin_mlp_int8_run(h, x, residual, y, residual_out, T, workspace, workspace_bytes, stream))


def swin_mlp_int8_run_debug(h, x, residual, y, residual_out, T, workspace, workspace_bytes, stream,
                            acc1, hidden, acc2, ln_out):
    _check(lib().swin_mlp_int8_run_debug(h, x, residual, y, residual_out, T, workspace, workspace_bytes,
                                         stream, acc1, hidden, acc2, ln_out))


def swin_mlp_int8_host_workspace_bytes(h, T, with_residual) -> int:
    return int(lib().swin_mlp_int8_host_workspace_bytes(h, T, int(with_residual)))


def swin_mlp_int8_run_host(h, x_host, residual_host, y_host, T, workspace, workspace_bytes, stream):
    _check(lib().swin_mlp_int8_run_host(h, x_host, residual_host, y_host, T, workspace, workspace_bytes, stream))


def _arrays(handles, xs, ys, Ts):
    n = len(handles)
    hv = (ctypes.c_void_p * n)(*[h for h in handles])
    xv = (ctypes.c_void_p * n)(*[0 if x is None else (x if isinstance(x, int) else x.data_ptr()) for x in xs]) \
        if xs is not None else None
    yv = (ctypes.c_void_p * n)(*[0 if y is None else (y if isinstance(y, int) else y.data_ptr()) for y in ys]) \
        if ys is not None else None
    tv = (ctypes.c_int64 * n)(*[int(t) for t in Ts])
    return n, hv, xv, yv, tv


def swin_mlp_int8_host_batch_workspace_bytes(handles, Ts) -> int:
    n, hv, _, _, tv = _arrays(handles, None, None, Ts)
    return int(lib().swin_mlp_int8_host_batch_workspace_bytes(n, hv, tv))


def swin_mlp_int8_run_host_batch(handles, x_hosts, y_hosts, Ts, workspace, workspace_bytes, stream):
    """x_hosts / y_hosts: pinned CPU tensors (or raw host pointers as ints)."""
    n, hv, xv, yv, tv = _arrays(handles, x_hosts, y_hosts, Ts)
    _check(lib().swin_mlp_int8_run_host_batch(n, hv, xv, yv, tv, workspace, workspace_bytes, stream))


def swin_mlp_int8_destroy(h):
    _check(lib().swin_mlp_int8_destroy(h))


def swin_mlp_int8_launches_per_run(h) -> int:
    return int(lib().swin_mlp_int8_launches_per_run(h))


def swin_mlp_int8_last_error() -> str:
    return last_error()


def swin_proj_int8_create(desc: swin_proj_int8_desc_t) -> int:
    h = ctypes.c_void_p()
    _check(lib().swin_proj_int8_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def swin_proj_int8_run(h, a, residual, y, residual_out, T, stream):
    _check(lib().swin_proj_int8_run(h, a, residual, y, residual_out, T, stream))


def swin_proj_int8_run_debug(h, a, residual, y, residual_out, T, stream, acc, ln_out):
    _check(lib().swin_proj_int8_run_debug(h, a, residual, y, residual_out, T, stream, acc, ln_out))


def swin_proj_int8_destroy(h):
    _check(lib().swin_proj_int8_destroy(h))


# ---- torch-facing convenience (device memory + streams only) ---------------------
def _ptr(t):
    return None if t is None else ctypes.c_void_p(t.data_ptr())


class SwinMlpInt8Layer:
    """One layer handle.  `layer` is any object with the fields of
    swin_mlp_int8_desc_t (e.g. synth.Layer); numpy arrays are passed as host
    pointers and copied by swin_mlp_int8_create."""

    def __init__(self, layer, device: int = 0, ln_fp64: bool = False, op5_unfused: bool = False):
        import numpy as np
        import torch
        self._keep = []

        def hp(a, dt):
            if a is None:
                return None
            if isinstance(a, torch.Tensor):      # host or device tensor: create() detects which
                a = a.contiguous()
                self._keep.append(a)
                return a.data_ptr()
            a = np.ascontiguousarray(a, dtype=dt)
            self._keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p).value

        d = swin_mlp_int8_desc_t()
        d.C, d.H, d.act = int(layer.C), int(layer.H), int(layer.act)
        d.x_scale, d.x_zero_point = float(layer.s_x), int(layer.z_x)
        d.w1, d.w1_scale, d.b1 = hp(layer.w1, np.int8), hp(layer.s_w1, np.float32), hp(layer.b1, np.float32)
        d.h_scale, d.h_zero_point = float(layer.s_h), int(layer.z_h)
        d.w2, d.w2_scale, d.b2 = hp(layer.w2, np.int8), hp(layer.s_w2, np.float32), hp(layer.b2, np.float32)
        d.ln_gamma, d.ln_beta, d.ln_eps = hp(layer.gamma, np.float32), hp(layer.beta, np.float32), float(layer.eps)
        d.y_scale, d.y_zero_point = float(layer.s_y), int(layer.z_y)
        d.device = int(device)
        d.ln_fp64 = int(bool(ln_fp64))
        d.op5_unfused = int(bool(op5_unfused))   # FT-style baseline: A1 through HBM, separate op #5
        d.gelu_in_scale = float(getattr(layer, "s_g", 0.0) or 0.0)   # shift-GELU control only
        self.C, self.H, self.device = d.C, d.H, device
        self.handle = swin_mlp_int8_create(d)
        self._keep = []
        self._ws = None
        self._torch = torch

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().swin_mlp_int8_destroy(h)
            except Exception:
                pass
            self.handle = None

    def plan(self, T=None):
        """The layer's launch plan; with T, the plans a run of T tokens launches."""
        out = (ctypes.c_int32 * 20)()
        if T is None:
            lib().swin_mlp_int8_plan(self.handle, out)
        elif lib().swin_mlp_int8_plan_for(self.handle, int(T), out) != 0:
            raise ValueError(f"swin_mlp_int8_plan_for: bad T = {T}")
        if out[12]:
            return {"fused": 1, "stages": out[13], "hq_buffers": out[14], "acc1_buffers": out[15],
                    "x_slots": out[17], "w2_stages": out[18],
                    "weights": "resident" if out[13] == 0 else "streamed"}
        return {"fused": 0, "fc1_bn": out[0], "fc1_cs": out[1], "fc1_stages": out[2], "fc1_max_clusters": out[3],
                "fc2_bn": out[4], "fc2_cs": out[5], "fc2_stages": out[6], "fc2_max_clusters": out[7],
                "fc1_groups": out[8], "fc2_groups": out[9], "fc1_resb": out[10], "fc2_resb": out[11],
                "fc1_pair": out[16], "op5_unfused": out[19] & 1,
                **({"run_plan": ("default", "ln_pair", "few_tile", "one_launch")[out[19] >> 1], "fc2_ksplit": out[13]}
                   if T is not None else {})}

    def set_plan_hint(self, T_hint=0):
        """Choose launch plans as for a run of T_hint tokens (0: per run); see the header."""
        _check(lib().swin_mlp_int8_set_plan_hint(self.handle, int(T_hint)))

    def set_trace(self, buf=None, cta=0):
        """buf: int64 device tensor of >= 9216 elements (see swin_mlp_int8_set_trace), or None."""
        _check(lib().swin_mlp_int8_set_trace(self.handle, _ptr(buf), int(cta)))

    def profile_begin(self, max_runs):
        _check(lib().swin_mlp_int8_profile_begin(self.handle, int(max_runs)))

    def profile_end(self):
        """Returns (fc1_ms_total, fc2_ms_total, runs) of the runs recorded since profile_begin."""
        a, b, n = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32()
        _check(lib().swin_mlp_int8_profile_end(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def constants(self):
        import numpy as np
        m1 = np.empty(self.H, np.float32); m2 = np.empty(self.C, np.float32)
        w1 = np.empty(self.H, np.int32); w2 = np.empty(self.C, np.int32)
        ih = ctypes.c_float(); iy = ctypes.c_float()
        P = lambda a: a.ctypes.data_as(ctypes.c_void_p)
        _check(lib().swin_mlp_int8_get_constants(self.handle, P(m1), ctypes.byref(ih), P(m2), ctypes.byref(iy),
                                                 P(w1), P(w2)))
        return m1, ih.value, m2, iy.value, w1, w2

    def workspace(self, T):
        torch = self._torch
        n = swin_mlp_int8_workspace_bytes(self.handle, T)
        if self._ws is None or self._ws.numel() < n:
            self._ws = torch.empty(max(n, 128), dtype=torch.uint8, device=f"cuda:{self.device}")
        return self._ws

    def __call__(self, x, residual=None, y=None, residual_out=None, stream=None, workspace=None):
        torch = self._torch
        T = x.shape[0]
        if y is None:
            y = torch.empty((T, self.C), dtype=torch.int8, device=x.device)
        ws = self.workspace(T) if workspace is None else workspace
        s = torch.cuda.current_stream(x.device).cuda_stream if stream is None else stream
        swin_mlp_int8_run(self.handle, _ptr(x), _ptr(residual), _ptr(y), _ptr(residual_out), T,
                          _ptr(ws), ws.numel(), ctypes.c_void_p(s))
        return y

    def run_debug(self, x, residual=None, residual_out=None):
        torch = self._torch
        T = x.shape[0]
        dev = x.device
        y = torch.empty((T, self.C), dtype=torch.int8, device=dev)
        acc1 = torch.empty((T, self.H), dtype=torch.int32, device=dev)
        hid = torch.empty((T, self.H), dtype=torch.int8, device=dev)
        acc2 = torch.empty((T, self.C), dtype=torch.int32, device=dev)
        ln = torch.empty((T, self.C), dtype=torch.float32, device=dev)
        ws = self.workspace(T)
        s = torch.cuda.current_stream(dev).cuda_stream
        swin_mlp_int8_run_debug(self.handle, _ptr(x), _ptr(residual), _ptr(y), _ptr(residual_out), T,
                                _ptr(ws), ws.numel(), ctypes.c_void_p(s),
                                _ptr(acc1), _ptr(hid), _ptr(acc2), _ptr(ln))
        return {"y": y, "acc1": acc1, "hidden": hid, "acc2": acc2, "yhat": ln}

    def run_host(self, x_host, y_host, residual_host=None, workspace=None, stream=None):
        """x_host/y_host/residual_host: pinned CPU tensors (host pointers into the C ABI)."""
        torch = self._torch
        T = x_host.shape[0]
        n = swin_mlp_int8_host_workspace_bytes(self.handle, T, residual_host is not None)
        ws = workspace if workspace is not None else torch.empty(n, dtype=torch.uint8, device=f"cuda:{self.device}")
        s = torch.cuda.current_stream(self.device).cuda_stream if stream is None else stream
        swin_mlp_int8_run_host(self.handle, _ptr(x_host), _ptr(residual_host), _ptr(y_host), T,
                               _ptr(ws), ws.numel(), ctypes.c_void_p(s))
        return y_host


class SwinProjInt8Layer:
    """Proj GEMM + fused op #4 (+ LN2) handle (include/swin_mlp_int8.h).
    `layer` has the fields of synth.ProjLayer (C, s_a, z_a, w, s_w, b, gamma, beta, eps, s_y, z_y)."""

    def __init__(self, layer, device: int = 0, ln_fp64: bool = False):
        import numpy as np
        import torch
        keep = []

        def hp(a, dt):
            if a is None:
                return None
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a.ctypes.data_as(ctypes.c_void_p).value

        d = swin_proj_int8_desc_t()
        d.C = int(layer.C)
        d.a_scale, d.a_zero_point = float(layer.s_a), int(layer.z_a)
        d.w, d.w_scale, d.b = hp(layer.w, np.int8), hp(layer.s_w, np.float32), hp(layer.b, np.float32)
        d.ln_gamma, d.ln_beta, d.ln_eps = hp(layer.gamma, np.float32), hp(layer.beta, np.float32), float(layer.eps)
        d.y_scale, d.y_zero_point = float(layer.s_y), int(layer.z_y)
        d.device, d.ln_fp64 = int(device), int(bool(ln_fp64))
        self.C, self.device = d.C, device
        self.handle = swin_proj_int8_create(d)
        self._torch = torch

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().swin_proj_int8_destroy(h)
            except Exception:
                pass
            self.handle = None

    def plan(self):
        out = (ctypes.c_int32 * 4)()
        lib().swin_proj_int8_plan(self.handle, out)
        return {"bn": out[0], "cs": out[1], "stages": out[2], "pair": out[3]}

    def __call__(self, a, residual, y=None, residual_out=None):
        torch = self._torch
        T = a.shape[0]
        if y is None:
            y = torch.empty((T, self.C), dtype=torch.int8, device=a.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
        swin_proj_int8_run(self.handle, _ptr(a), _ptr(residual), _ptr(y), _ptr(residual_out), T, stream)
        return y

    def run_debug(self, a, residual, residual_out=None):
        torch = self._torch
        T = a.shape[0]
        y = torch.empty((T, self.C), dtype=torch.int8, device=a.device)
        acc = torch.empty((T, self.C), dtype=torch.int32, device=a.device)
        ln = torch.empty((T, self.C), dtype=torch.float32, device=a.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(a.device).cuda_stream)
        swin_proj_int8_run_debug(self.handle, _ptr(a), _ptr(residual), _ptr(y), _ptr(residual_out), T, stream,
                                 _ptr(acc), _ptr(ln))
        return {"y": y, "acc": acc, "ln_out": ln}


# ---- attention half (include/swin_attn_int8.h) -------------------

def swin_op1_int8_create(desc: swin_op1_int8_desc_t) -> int:
    h = ctypes.c_void_p()
    _check(lib().swin_op1_int8_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def swin_op1_int8_run(h, x, B, y, stream):
    _check(lib().swin_op1_int8_run(h, x, B, y, stream))


def swin_op1_int8_destroy(h):
    _check(lib().swin_op1_int8_destroy(h))


def swin_attn_int8_create(desc: swin_attn_int8_desc_t) -> int:
    h = ctypes.c_void_p()
    _check(lib().swin_attn_int8_create(ctypes.byref(desc), ctypes.byref(h)))
    return h.value


def swin_attn_int8_workspace_bytes(h, B) -> int:
    return int(lib().swin_attn_int8_workspace_bytes(h, B))


def swin_attn_int8_run(h, xw, B, a, workspace, workspace_bytes, stream):
    _check(lib().swin_attn_int8_run(h, xw, B, a, workspace, workspace_bytes, stream))


def swin_attn_int8_run_debug(h, xw, B, a, workspace, workspace_bytes, stream, qkv, acc, p):
    _check(lib().swin_attn_int8_run_debug(h, xw, B, a, workspace, workspace_bytes, stream, qkv, acc, p))


def swin_attn_int8_destroy(h):
    _check(lib().swin_attn_int8_destroy(h))


def _host_ptr(keep, a, dt):
    import numpy as np
    if a is None:
        return None
    a = np.ascontiguousarray(a, dtype=dt)
    keep.append(a)
    return a.ctypes.data_as(ctypes.c_void_p).value


class SwinOp1Int8:
    """Fused op #1 handle (LayerNorm -> window shift -> Q).  `layer`: synth.AttnLayer (or any
    object with C, M, shift, Hs, Ws, gamma1, beta1, eps, s_x, z_x)."""

    def __init__(self, layer, device: int = 0):
        import numpy as np
        import torch
        keep = []
        d = swin_op1_int8_desc_t()
        d.C, d.M, d.shift, d.Hs, d.Ws = int(layer.C), int(layer.M), int(layer.shift), int(layer.Hs), int(layer.Ws)
        d.ln_gamma, d.ln_beta = _host_ptr(keep, layer.gamma1, np.float32), _host_ptr(keep, layer.beta1, np.float32)
        d.ln_eps, d.y_scale, d.y_zero_point, d.device = float(layer.eps), float(layer.s_x), int(layer.z_x), int(device)
        self.C, self.Hs, self.Ws = d.C, d.Hs, d.Ws
        self.handle = swin_op1_int8_create(d)
        self._torch = torch

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().swin_op1_int8_destroy(h)
            except Exception:
                pass
            self.handle = None

    def __call__(self, x, y=None):
        """x: fp32 [B][Hs][Ws][C] device tensor -> int8 [B*Hs*Ws][C] (window order)."""
        torch = self._torch
        B = x.shape[0]
        if y is None:
            y = torch.empty((B * self.Hs * self.Ws, self.C), dtype=torch.int8, device=x.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(x.device).cuda_stream)
        swin_op1_int8_run(self.handle, _ptr(x), B, _ptr(y), stream)
        return y


class SwinAttnInt8Layer:
    """QKV GEMM + op #2 -> Q.K + op #3 -> V.att handle.  `layer`: synth.AttnLayer."""

    def __init__(self, layer, device: int = 0):
        import numpy as np
        import torch
        keep = []
        d = swin_attn_int8_desc_t()
        d.C, d.heads, d.M, d.shift = int(layer.C), int(layer.heads), int(layer.M), int(layer.shift)
        d.Hs, d.Ws = int(layer.Hs), int(layer.Ws)
        d.x_scale, d.x_zero_point = float(layer.s_x), int(layer.z_x)
        d.w_qkv = _host_ptr(keep, layer.w_qkv, np.int8)
        d.w_qkv_scale = _host_ptr(keep, layer.s_wqkv, np.float32)
        d.b_qkv = _host_ptr(keep, layer.b_qkv, np.float32)
        d.q_scale, d.k_scale, d.v_scale = float(layer.s_q), float(layer.s_k), float(layer.s_v)
        d.rel_bias_table = _host_ptr(keep, layer.table, np.float32)
        d.a_scale, d.a_zero_point, d.device = float(layer.s_a), int(layer.z_a), int(device)
        self.C, self.heads, self.M, self.Hs, self.Ws = d.C, d.heads, d.M, d.Hs, d.Ws
        self.handle = swin_attn_int8_create(d)
        self._torch = torch
        self._ws = None

    def __del__(self):
        h = getattr(self, "handle", None)
        if h:
            try:
                lib().swin_attn_int8_destroy(h)
            except Exception:
                pass
            self.handle = None

    def workspace(self, B, device=None):
        n = max(swin_attn_int8_workspace_bytes(self.handle, B), 128)
        if self._ws is None or self._ws.numel() < n:
            self._ws = self._torch.empty(n, dtype=self._torch.uint8, device=device or "cuda")
        return self._ws

    def constants(self):
        import numpy as np
        c = np.empty(3, np.float32)
        N = self.M * self.M
        bias = np.empty((self.heads, N, N), np.float32)
        _check(lib().swin_attn_int8_get_constants(self.handle, c.ctypes.data_as(ctypes.c_void_p),
                                                  bias.ctypes.data_as(ctypes.c_void_p)))
        return {"m3": float(c[0]), "inv_p": float(c[1]), "m_o": float(c[2]), "bias": bias}

    def __call__(self, xw, B, a=None, workspace=None):
        """xw: int8 [B*Hs*Ws][C] window order (op #1's output) -> int8 [B*Hs*Ws][C] raster order."""
        torch = self._torch
        T = xw.shape[0]
        if a is None:
            a = torch.empty((T, self.C), dtype=torch.int8, device=xw.device)
        ws = workspace if workspace is not None else self.workspace(B, xw.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(xw.device).cuda_stream)
        swin_attn_int8_run(self.handle, _ptr(xw), B, _ptr(a), _ptr(ws), ws.numel(), stream)
        return a

    def profile_begin(self, max_runs):
        _check(lib().swin_attn_int8_profile_begin(self.handle, int(max_runs)))

    def profile_end(self):
        """(qkv_gemm_ms_total, core_ms_total, runs) of the runs recorded since profile_begin."""
        a, b, n = ctypes.c_float(), ctypes.c_float(), ctypes.c_int32()
        _check(lib().swin_attn_int8_profile_end(self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(n)))
        return a.value, b.value, n.value

    def run_debug(self, xw, B):
        torch = self._torch
        T = xw.shape[0]
        N = self.M * self.M
        a = torch.empty((T, self.C), dtype=torch.int8, device=xw.device)
        qkv = torch.empty((T, 3 * self.C), dtype=torch.int8, device=xw.device)
        acc = torch.empty((T, 3 * self.C), dtype=torch.int32, device=xw.device)
        p = torch.empty((T // N, self.heads, N, N), dtype=torch.int8, device=xw.device)
        ws = self.workspace(B, xw.device)
        stream = ctypes.c_void_p(torch.cuda.current_stream(xw.device).cuda_stream)
        swin_attn_int8_run_debug(self.handle, _ptr(xw), B, _ptr(a), _ptr(ws), ws.numel(), stream,
                                 _ptr(qkv), _ptr(acc), _ptr(p))
        return {"a": a, "qkv": qkv, "acc": acc, "p": p}
