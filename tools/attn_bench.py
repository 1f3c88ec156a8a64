"""Attention half of the Swin block at the BASELINE shapes: fused
op #1 (LayerNorm -> window shift -> Q), the QKV GEMM + op #2 and the window-attention core (Q.K ->
op #3 -> V.att), each timed with CUDA events on the launching stream, L2 flushed before every run.
Rooflines: op #1 and the core are HBM-bound (algorithmic bytes 5C and 4C per token), the QKV GEMM
against the int8 tensor roof (6 C^2 ops per token).

usage: python tools/attn_bench.py [swin_t|swin_b|swin_l] [--steps K]   -> one JSON line per stage"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2402_01169_b200 import SwinAttnInt8Layer, SwinMlpInt8Layer, SwinOp1Int8, SwinProjInt8Layer  # noqa: E402

# (name, batch, C0, img, window): the per-GPU shapes of BASELINE configs[1], [3] (b128 per GPU), [4]
MODELS = {"swin_t": ("Swin-T b64", 64, 96, 224, 7), "swin_b": ("Swin-B b128", 128, 128, 224, 7),
          "swin_l": ("Swin-L 384 b64", 64, 192, 384, 12)}


def peaks():
    d = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    return d["hbm_gbs"], 2.0 * d["bf16_tflops"]


def run(model="swin_t", steps=20):
    name, B, C0, img, M = MODELS[model]
    hbm, int8_peak = peaks()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for s in range(4):
        C, S = C0 << s, img // 4 >> s
        shift = M // 2 if S > M else 0   # (the shifted block of the stage; none when one window covers it)
        A = synth.make_attn_layer(C, S, S, synth.layer_seed(9, s, 0), M=M, shift=shift)
        op1, attn = SwinOp1Int8(A, device=0), SwinAttnInt8Layer(A, device=0)
        x = torch.from_numpy(synth.make_block_input(B, S, S, C, 11 + s)).cuda()
        T = B * S * S
        xw = torch.empty((T, C), dtype=torch.int8, device="cuda")
        a = torch.empty((T, C), dtype=torch.int8, device="cuda")
        ws = attn.workspace(B)
        for _ in range(3):
            op1(x, y=xw)
            attn(xw, B, a=a, workspace=ws)
        torch.cuda.synchronize()

        def timed(fn):
            ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
            for k in range(steps):
                flush.fill_(k & 0xff)
                ev[k][0].record()
                fn()
                ev[k][1].record()
            torch.cuda.synchronize()
            v = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)
            return v[len(v) // 2]

        us_op1 = timed(lambda: op1(x, y=xw))
        us_attn = timed(lambda: attn(xw, B, a=a, workspace=ws))
        # the rest of the block: Proj + op #4 (+LN2) on the residual stream, then the MLP (ReLU)
        P = synth.make_proj(C, synth.layer_seed(9, s, 1))
        P.s_a, P.z_a = A.s_a, A.z_a
        Lm = synth.make_layer(C, synth.layer_seed(9, s, 2))
        Lm.s_x, Lm.z_x = P.s_y, P.z_y
        proj, mlp = SwinProjInt8Layer(P, device=0), SwinMlpInt8Layer(Lm, device=0)
        R = x.reshape(T, C)
        zb = torch.empty((T, C), dtype=torch.float32, device="cuda")
        y4 = torch.empty((T, C), dtype=torch.int8, device="cuda")
        yb = torch.empty((T, C), dtype=torch.int8, device="cuda")
        mws = torch.empty(max(mlp.workspace(T).numel(), 128), dtype=torch.uint8, device="cuda")

        def block():
            op1(x, y=xw)
            attn(xw, B, a=a, workspace=ws)
            proj(a, R, y=y4, residual_out=zb)
            mlp(y4, y=yb, residual=zb, workspace=mws)

        for _ in range(2):
            block()
        torch.cuda.synchronize()
        us_block = timed(block)
        attn.profile_begin(steps)
        for k in range(steps):
            flush.fill_(k & 0xff)
            attn(xw, B, a=a, workspace=ws)
        torch.cuda.synchronize()
        q_ms, c_ms, n = attn.profile_end()
        us_qkv, us_core = 1e3 * q_ms / max(n, 1), 1e3 * c_ms / max(n, 1)
        N = M * M
        b_op1, b_core = 5.0 * C * T, 4.0 * C * T
        ops_qkv = 2.0 * T * C * 3 * C
        rows.append({"model": name, "stage": s, "C": C, "T": T, "heads": C // 32, "window": M, "shift": shift,
                     "op1_us": round(us_op1, 2), "op1_gbs": round(b_op1 / us_op1 / 1e3, 1),
                     "op1_hbm_frac": round(b_op1 / us_op1 / 1e3 / hbm, 3),
                     "attn_us": round(us_attn, 2), "qkv_us": round(us_qkv, 2), "core_us": round(us_core, 2),
                     "qkv_tops": round(ops_qkv / us_qkv / 1e6, 1), "qkv_tensor_frac": round(ops_qkv / us_qkv / 1e6 / int8_peak, 3),
                     "core_gbs": round(b_core / us_core / 1e3, 1), "core_hbm_frac": round(b_core / us_core / 1e3 / hbm, 3),
                     "core_gops": round(4.0 * N * C * T / us_core / 1e3, 1),
                     "tokens_per_s_attn_half": T / ((us_op1 + us_attn) * 1e-6),
                     "block_us": round(us_block, 2), "block_tokens_per_s": T / (us_block * 1e-6),
                     "block": "op #1 -> QKV/op #2 -> attention core -> Proj/op #4 (+LN2) -> MLP (ReLU), 7 launches"})
        del op1, attn, x, xw, a, proj, mlp
        torch.cuda.empty_cache()
    return {"what": "attention half: op #1 + QKV GEMM/op #2 + attention core (NEXT-4 / NEXT-3), and the whole block",
            "bytes_per_token": {"op1": "4C read (fp32) + C write", "core": "3C read (qkv) + C write"},
            "hbm_peak_gbs": hbm, "int8_peak_tops": int8_peak, "l2": "flushed before every run", "rows": rows}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("models", nargs="*", default=["swin_t"])
    ap.add_argument("--steps", type=int, default=20)
    a = ap.parse_args()
    for m in a.models:
        print(json.dumps(run(m, a.steps)), flush=True)
