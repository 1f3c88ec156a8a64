"""Whole MLP stacks of BASELINE configs 3-5 on ONE B200 (the per-GPU share of the token-sharded
multi-GPU runs): every layer of every stage, layer l of a stage feeding layer l+1 (SURVEY.md
§8(d) recipe), L2 flushed before each timed step, CUDA events on the launching stream.

  config 3  Swin-S, batch 256 (1 GPU: the whole batch; --batch to shard)
  config 4  Swin-B, batch 1024 / 8 GPUs = 128 per GPU   (the north star's >= 60 % target)
  config 5  Swin-L 384x384 (window 12), batch 512 / 8 = 64 per GPU

usage: python tools/stack_bench.py [config ...] [--steps K] [--act relu|gelu] [--json FILE]
Prints one JSON line per config (tokens/s, ms/step, TOPS and the fraction of the int8
tensor roof, per-stage kernel times from native per-kernel events)."""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402
from paper_2402_01169_b200 import SwinMlpInt8Layer, swin_mlp_int8_workspace_bytes  # noqa: E402

PER_GPU_BATCH = {3: 256, 4: 1024 // 8, 5: 512 // 8}
NAME = {3: "Swin-S b256", 4: "Swin-B b1024 (per GPU of 8: b128)", 5: "Swin-L 384 b512 (per GPU of 8: b64)"}


def int8_peak_tops():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return 2.0 * json.load(open(p))["bf16_tflops"], "MEASURED_PEAKS.json bf16 x 2"
    return 2.0 * 1590.0, "B200_PROFILING.md fallback bf16 x 2"


def run(config, steps, act, op5_unfused=False):
    batch = PER_GPU_BATCH[config]
    stages = synth.config_layers(config, batch=batch)
    layers = []   # (layer handle, stage, T, C)
    bufs, ws = [], 0
    for s, (C, T, n) in enumerate(stages):
        X = synth.make_activations(synth.make_layer(C, synth.layer_seed(config, s, 0), act=act), T,
                                   synth.layer_seed(config, s, 0) + 50)
        a = torch.from_numpy(X).cuda()
        b = torch.empty_like(a)
        bufs.append((a, b))
        for l in range(n):
            L = synth.make_layer(C, synth.layer_seed(config, s, l), act=act)
            h = SwinMlpInt8Layer(L, device=0, op5_unfused=op5_unfused)
            layers.append((h, s, l, T, C))
            ws = max(ws, swin_mlp_int8_workspace_bytes(h.handle, T))
    work = torch.empty(max(ws, 128), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def step():
        for h, s, l, T, C in layers:
            a, b = bufs[s]
            x, y = (a, b) if l % 2 == 0 else (b, a)
            h(x, y=y, workspace=work)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.fill_(k & 0xff)
        ev[k][0].record()
        step()
        ev[k][1].record()
    torch.cuda.synchronize()
    ms = sorted(a.elapsed_time(b) for a, b in ev)
    t = sum(ms) / steps
    # per-kernel times (a second pass with native events around every kernel)
    for h, *_ in layers:
        h.profile_begin(steps)
    for k in range(steps):
        flush.fill_(k & 0xff)
        step()
    torch.cuda.synchronize()
    per_stage = {}
    for (h, s, l, T, C) in layers:
        f1, f2, n = h.profile_end()
        per_stage.setdefault(s, [0.0, 0, T, C, h.plan().get("fused", 0)])
        per_stage[s][0] += (f1 + f2) / max(n, 1) * 1e3
        per_stage[s][1] += 1
    tokens = sum(T for _, _, _, T, _ in layers)
    ops = sum(16.0 * C * C * T for _, _, _, T, C in layers)
    peak, src = int8_peak_tops()
    tops = ops / (t / 1e3) / 1e12
    return {"config": config, "workload": NAME[config], "act": act_name(act), "op5_unfused": op5_unfused,
            "layers": len(layers), "ms_per_step": t, "ms_median": ms[len(ms) // 2],
            "tokens_per_s": tokens / (t / 1e3), "layer_tokens_per_step": tokens, "tops": tops,
            "int8_peak_tops": peak, "peak_source": src, "tensor_frac": tops / peak,
            "stages": [{"C": v[3], "T": v[2], "layers": v[1], "fused": v[4], "profiled_us": round(v[0], 1),
                        "profiled_us_per_layer": round(v[0] / v[1], 2)} for _, v in sorted(per_stage.items())],
            "l2": "flushed between steps", "steps": steps}


def act_name(a):
    return "relu" if a == synth.ACT_RELU else "gelu"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="*", type=int, default=[3, 4, 5])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--act", default="relu", choices=["relu", "gelu"])
    ap.add_argument("--unfused", action="store_true", help="FasterTransformer-layout op #5 (NEXT-1)")
    ap.add_argument("--json", default=None)
    a = ap.parse_args()
    act = synth.ACT_RELU if a.act == "relu" else synth.ACT_GELU
    out = []
    for c in a.configs:
        r = run(c, a.steps, act, a.unfused)
        print(json.dumps(r), flush=True)
        out.append(r)
        torch.cuda.empty_cache()
    if a.json:
        json.dump(out, open(a.json, "w"), indent=1)


if __name__ == "__main__":
    main()
