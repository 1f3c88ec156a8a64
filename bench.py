"""Benchmark of the B200-native GELU-less INT8 Swin MLP sub-layer.

`python bench.py --gpus N --steps K --warmup W [--impl reference]`

Workload (BASELINE.json configs[1], the configuration the metric is quoted on
that fits one GPU): Swin-T, all four stage MLPs (C = 96/192/384/768, H = 4C)
at batch 64 -> T = 200704 / 50176 / 12544 / 3136 tokens.  One step = one pass
of the whole hot path (FC1 -> op #5 ReLU -> FC2 -> op #6 LN+Q) over all four
layers.  Multi-GPU: one process per GPU (torchrun), weights broadcast once from
rank 0 over NCCL, every rank runs its own batch of 64 images (weak scaling, no
collective on the hot path).  L2 is flushed (256 MiB write, untimed) before
every timed step; each step is timed with CUDA events on the launching stream;
the job time is the max over ranks.

Rank 0 prints ONE JSON line (see README/DESIGN.md §6 for every key).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s per Swin MLP layer at 1/2/4/8 B200; % INT8 TC peak; ReLU vs GELU us"
WORKLOAD = ("configs[1]: Swin-T all four stage MLPs (C=96/192/384/768 -> 4C -> C; "
            "T=200704/50176/12544/3136 tokens), batch 64 per GPU, int8")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--pairs", type=int, default=30, help="interleaved ReLU/GELU paired trials")
    ap.add_argument("--cpu-stride", type=int, default=1, help="cpu_baseline samples every n-th token")
    ap.add_argument("--ref-stride", type=int, default=64, help="--impl reference samples every n-th token")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-stack", action="store_true", help="skip the Swin-B stack (north star) measurement")
    return ap.parse_args()


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def layers_spec(batch, act):
    import synth
    toks = synth.stage_tokens(batch)
    out = []
    for s in range(4):
        C = 96 << s
        out.append((synth.make_layer(C, synth.layer_seed(2, s, 0), act=act), toks[s], synth.layer_seed(2, s, 0) + 50))
    return out


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16_burst": d["bf16_tflops"], "bf16_sustained": d.get("bf16_tflops_sustained"),
                "hbm_gbs": d["hbm_gbs"], "src": "MEASURED_PEAKS.json", "sm_max_mhz": d.get("sm_max_mhz")}
    return {"bf16_burst": 1590.0, "bf16_sustained": 1400.0, "hbm_gbs": 6650.0,
            "src": "B200_PROFILING.md fallback", "sm_max_mhz": 1965.0}


class ClockSampler:
    """NVML SM-clock / throttle-reason sampling during the timed region."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, index, period=0.002):
        self.samples, self.reasons, self.period = [], set(), period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self.nv = None
            self.max = None

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.nv:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.nv:
            self._stop.set()
            self.t.join()

    def result(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def cpu_oracle_rate(spec, stride, offset=0, nthreads=0):
    """Oracle tokens/s on every `stride`-th token of each layer (bounded sample)."""
    import numpy as np
    import oracle
    import synth
    nthreads = nthreads or os.cpu_count()
    tok = 0
    t_total = 0.0
    for L, T, xs in spec:
        X = synth.make_activations(L, T, xs)
        rows = np.arange(offset % stride, T, stride, dtype=np.int64)
        t0 = time.perf_counter()
        oracle.mlp(L, X, rows=rows, nthreads=nthreads)
        t_total += time.perf_counter() - t0
        tok += rows.size
    return tok / t_total, tok, t_total, nthreads


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def oracle_per_c_table():
    """SURVEY.md §8(d) oracle timing: tokens/s of the oracle as it stands per distinct C, on 2048
    rows with every host core and on 128 rows with one thread (cost is linear in T)."""
    import numpy as np
    import oracle
    import synth
    out = []
    for C in (96, 192, 384, 768):
        L = synth.make_layer(C, synth.layer_seed(2, 0, 0) + C)
        X = synth.make_activations(L, 2048, 5)
        row = {"C": C}
        for key, n, nth in (("all_cores", 2048, os.cpu_count()), ("one_thread", 128, 1)):
            t0 = time.perf_counter()
            oracle.mlp(L, X, rows=np.arange(n, dtype=np.int64), nthreads=nth)
            row[key + "_tokens_per_s"] = n / (time.perf_counter() - t0)
        out.append(row)
    return out


def run_reference(args, ws, rank):
    """--impl reference: the oracle as it stands on the host cores (rank 0 only)."""
    if rank != 0:
        return
    import synth
    spec = layers_spec(args.batch, synth.ACT_RELU)
    total_tok, total_t = 0, 0.0
    for i in range(args.warmup):
        cpu_oracle_rate(spec, args.ref_stride * 4, offset=i)
    nth = os.cpu_count()
    for k in range(args.steps):
        _, tok, t, nth = cpu_oracle_rate(spec, args.ref_stride, offset=k)
        total_tok += tok
        total_t += t
    v = total_tok / total_t
    sample = f"every {args.ref_stride}th token of each of the 4 layers per step ({total_tok // max(1, args.steps)} tokens/step)"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total_t / args.steps,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "s8",
            "data": "synthetic", "config": {"workload": WORKLOAD, "sample": sample},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": nth, "kind": "oracle", "sample": sample},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def refuse_plan_switches():
    """The library reads SWIN_MLP_* A/B switches (plan variants, PDL off, sync checks) at create
    time; a bench number taken under any of them is not the product's, so refuse to run."""
    bad = sorted(k for k in os.environ if k.startswith("SWIN_MLP_"))
    if bad:
        raise SystemExit(f"bench.py: refusing to run with plan/debug switches set: {', '.join(bad)}")


def main():
    args = parse()
    refuse_plan_switches()
    ws, rank, local = dist_env()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import synth
    import paper_2402_01169_b200 as P
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    from paper_2402_01169_b200.dist import broadcast_layer

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    P.lib()

    # ---- layers: rank 0 generates, weights broadcast once over NCCL --------------------------------
    spec = layers_spec(args.batch, synth.ACT_RELU)
    relu_layers, gelu_layers, xs_dev, xs_host, ys, T_list = [], [], [], [], [], []
    ft_gelu_layers, ft_relu_layers = [], []   # FasterTransformer layout: op #5 unfused (NEXT-1)
    sg_layers = []   # the I-ViT shift-GELU control (NEXT-4; always unfused: it needs each row's max)
    for li, (L, T, xseed) in enumerate(spec):
        if ws > 1:
            broadcast_layer(L, dev)   # create() copies from the device tensors
        relu_layers.append(SwinMlpInt8Layer(L, device=local))
        ft_relu_layers.append(SwinMlpInt8Layer(L, device=local, op5_unfused=True))
        L.act = synth.ACT_GELU
        gelu_layers.append(SwinMlpInt8Layer(L, device=local))
        ft_gelu_layers.append(SwinMlpInt8Layer(L, device=local, op5_unfused=True))
        L.act = synth.ACT_SHIFT_GELU
        sg_layers.append(SwinMlpInt8Layer(L, device=local))
        L.act = synth.ACT_RELU
        X = synth.make_activations(L, T, xseed + 7919 * rank)
        xh = torch.from_numpy(X).pin_memory()
        xs_host.append(xh)
        xs_dev.append(xh.to(dev))
        ys.append(torch.empty((T, L.C), dtype=torch.int8, device=dev))
        T_list.append(T)
    ws_bytes = max(P.swin_mlp_int8_workspace_bytes(l.handle, T) for l, T in zip(ft_gelu_layers, T_list))
    host_ws = max(P.swin_mlp_int8_host_workspace_bytes(l.handle, T, 0) for l, T in zip(relu_layers, T_list))
    workspace = torch.empty(max(ws_bytes, host_ws), dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)
    tokens_per_step = sum(T_list)

    def step(layers):
        for l, x, y in zip(layers, xs_dev, ys):
            l(x, y=y, workspace=workspace)

    def timed(fn, n, flush_l2=True):
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(n)]
        for k in range(n):
            if flush_l2:
                flush.fill_(k & 0xff)
            evs[k][0].record(stream)
            fn()
            evs[k][1].record(stream)
        torch.cuda.synchronize(dev)
        return [a.elapsed_time(b) for a, b in evs]

    def barrier():
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize(dev)

    def max_over_ranks(v):
        if ws == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # ---- warm-up ---------------------------------------------------------------------------------
    for _ in range(max(args.warmup, 0)):
        step(relu_layers)
    torch.cuda.synchronize(dev)
    # guard against timing a no-op: every layer's output must be a live LayerNorm
    # output (non-constant rows, spread over the int8 grid); parity itself is the
    # tests' job (tests/test_parity_gpu.py), not the bench's
    for (L, T, _), y in zip(spec, ys):
        yf = y[: min(T, 4096)].float()
        if not (yf.std(dim=1).min().item() > 1.0 and yf.abs().max().item() > 16):
            raise RuntimeError(f"layer C={L.C}: output looks dead (kernel not executed?)")

    # ---- timed region: exactly K steps --------------------------------------------------------------
    # (step-boundary events only: events between the kernels of a step would serialise the
    # programmatic dependent launches that overlap one kernel's prologue with the previous
    # kernel's tail)
    sampler = ClockSampler(local)
    barrier()
    with sampler:
        per_step = timed(lambda: step(relu_layers), args.steps)
    barrier()
    t_ms = max_over_ranks(sum(per_step))
    value = ws * tokens_per_step * args.steps / (t_ms / 1e3)

    # ---- per-kernel durations: a second timed region of K identical steps with native CUDA
    # events around every kernel (swin_mlp_int8_profile_begin/end, on the launching stream)
    for l in relu_layers:
        l.profile_begin(args.steps)
    barrier()
    per_step_prof = timed(lambda: step(relu_layers), args.steps)
    barrier()
    prof = [l.profile_end() for l in relu_layers]

    # ---- roofline of the dominant kernel (per-launch CUDA events, native) -------------------------
    peaks = load_peaks()
    int8_peak_tops = 2.0 * peaks["bf16_burst"]      # nominal int8/bf16 dense ratio 4.5/2.25 = 2
    kernels = []
    for (L, T, _), (f1, f2, n), l in zip(spec, prof, relu_layers):
        ops = 2.0 * T * L.C * L.H
        e5, e6 = T * L.H * 3.5, T * L.C * 15.0     # algorithmic epilogue lane-instructions
        if l.plan()["fused"]:
            parts = (("fused_mlp", f1 + f2, 2.0 * ops, e5 + e6),)
        else:
            parts = (("fc1_relu_q", f1, ops, e5), ("fc2_ln_q", f2, ops, e6))
        for name, ms, kops, alu in parts:
            avg_s = ms / max(n, 1) / 1e3
            kernels.append({"kernel": f"{name}[C={L.C},T={T}]", "avg_us": avg_s * 1e6,
                            "tops": kops / avg_s / 1e12 if avg_s > 0 else None, "ops": kops, "alu": alu})
    dom = max(kernels, key=lambda k: k["avg_us"])
    step_us = 1e3 * sum(per_step_prof) / args.steps    # the profiled pass's own step time
    share = dom["avg_us"] / step_us
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        try:
            traffic = json.load(open(tpath)).get(dom["kernel"])
        except Exception:
            traffic = None
    # The binding roof of the dominant kernel: tensor (algorithmic int8 ops) or ALU (the
    # epilogues' algorithmic fp32 lane-instructions: e5 = 3.5 per hidden value
    # for ReLU op #5, e6 = 15 per output value for op #6, against 148 SMs x 128 lanes x the
    # max SM clock) -- whichever the kernel is closer to
    sm_hz = 1e6 * (peaks.get("sm_max_mhz") or 1965.0)
    alu_peak = 148 * 128 * sm_hz / 1e12          # T lane-instr/s
    tensor_view = {"bound": "tensor", "achieved": dom["tops"], "peak": int8_peak_tops, "unit": "TOPS",
                   "frac": dom["tops"] / int8_peak_tops,
                   "algorithmic": "2*T*C*H ops per GEMM per launch (fused_mlp: both GEMMs, 4*T*C*H); "
                                  "SURVEY §8(d): 16*C^2 ops per token per layer",
                   "peak_source": f"{peaks['src']} bf16_tflops {peaks['bf16_burst']} x 2 (int8:bf16 nominal 4.5:2.25), burst"}
    alu_ach = dom["alu"] / (dom["avg_us"] / 1e6) / 1e12
    alu_view = {"bound": "alu", "achieved": alu_ach, "peak": alu_peak, "unit": "T lane-instr/s",
                "frac": alu_ach / alu_peak,
                "algorithmic": "T*(H*3.5 + C*15) lane-instructions per layer (SURVEY §8(d) e5, e6); op #5 only "
                               "for fc1_relu_q, op #6 only for fc2_ln_q",
                "peak_source": "148 SMs x 128 fp32 lanes x max SM clock (B200_PROFILING / MEASURED_PEAKS)"}
    bind, other = (alu_view, tensor_view) if alu_view["frac"] > tensor_view["frac"] else (tensor_view, alu_view)
    roofline = {"bound": bind["bound"], "kernel": dom["kernel"], "achieved": bind["achieved"], "peak": bind["peak"],
                "unit": bind["unit"], "frac": bind["frac"], "traffic": traffic,
                "share_of_step": share,
                "peak_source": bind["peak_source"], "algorithmic": bind["algorithmic"],
                "other_roof": other,
                "step_frac": (sum(k["ops"] for k in kernels) / (t_ms / args.steps / 1e3) / 1e12) / int8_peak_tops,
                "profiled_step_us": step_us,
                "kernels": [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in kk.items()
                             if k not in ("ops", "alu")} for kk in kernels]}

    # ---- end to end through the C ABI with host buffers (H2D + run + D2H per step) ----------------
    # the user call for a step of the four independent stage MLPs: swin_mlp_int8_run_host_batch
    # (one copy-in / kernels / copy-out pipeline over all their token chunks); the per-layer
    # swin_mlp_int8_run_host loop is reported beside it
    ys_host = [torch.empty((T, L.C), dtype=torch.int8).pin_memory() for (L, T, _) in spec]
    hs = [l.handle for l in relu_layers]
    bws = P.swin_mlp_int8_host_batch_workspace_bytes(hs, T_list)
    bwork = torch.empty(bws, dtype=torch.uint8, device=dev)

    def step_host_batch():
        P.swin_mlp_int8_run_host_batch(hs, xs_host, ys_host, T_list, bwork.data_ptr(), bws, stream.cuda_stream)

    def step_host():
        for l, xh, yh in zip(relu_layers, xs_host, ys_host):
            l.run_host(xh, yh, workspace=workspace)

    e2e_steps = max(3, min(args.steps, 20))
    res_e2e = {}
    for name, fn in (("batch", step_host_batch), ("per_layer", step_host)):
        for _ in range(2):
            fn()
        barrier()
        ms = max_over_ranks(sum(timed(fn, e2e_steps)))
        barrier()
        res_e2e[name] = ws * tokens_per_step * e2e_steps / (ms / 1e3)
    e2e_val = res_e2e["batch"]
    h2d = sum(int(x.numel()) for x in xs_host)
    d2h = sum(int(y.numel()) for y in ys_host)

    # ---- ReLU vs GELU: interleaved trials of four arms, order rotated per trial --------------------
    #   relu     the GELU-less layer, ReLU folded into FC1's drain (the product)
    #   gelu     the same kernels with the exact-erf GELU epilogue (control)
    #   gelu_ft  the paper's baseline layout: FC1 -> A1 int32 in HBM -> separate dQ/GELU/Q kernel
    #            -> FC2 (FasterTransformer)
    #   relu_ft  the same unfused layout with ReLU (separates the fusion gain from the activation)
    #   shift_gelu the I-ViT integer shift-GELU (the paper's other comparison):
    #            FC1 -> A1 -> the row-max op #5 kernel -> FC2 (R28)
    arms = {"relu": relu_layers, "gelu": gelu_layers, "gelu_ft": ft_gelu_layers, "relu_ft": ft_relu_layers,
            "shift_gelu": sg_layers}
    for layers in arms.values():
        for _ in range(3):
            step(layers)
    samples = {k: [] for k in arms}
    wins = 0
    names = list(arms)
    for i in range(args.pairs):
        res = {}
        for k in names[i % len(names):] + names[:i % len(names)]:
            res[k] = 1e3 * timed(lambda: step(arms[k]), 1)[0]
        for k in names:
            samples[k].append(res[k])
        wins += res["relu"] < min(res["gelu"], res["gelu_ft"])
    med = {k: statistics.median(v) for k, v in samples.items()}
    relu_gelu = {"relu_us_median": med["relu"], "gelu_us_median": med["gelu"],
                 "gelu_over_relu": med["gelu"] / med["relu"],
                 "gelu_ft_us_median": med["gelu_ft"], "relu_ft_us_median": med["relu_ft"],
                 "shift_gelu_us_median": med["shift_gelu"],
                 "latency_gain_vs_shift_gelu": 1.0 - med["relu"] / med["shift_gelu"],
                 "latency_gain_vs_ft_gelu": 1.0 - med["relu"] / med["gelu_ft"],
                 "latency_gain_vs_fused_gelu": 1.0 - med["relu"] / med["gelu"],
                 "paper_context": "RTX 4090, whole Swin model: >= 11% latency gain from GELU->ReLU (PAPER.md:13)",
                 "pairs": args.pairs, "relu_wins": wins, "b1": "None in every arm (paper mode)",
                 "unit": "us per step (4 layers)"}

    # ---- the north star's stack (BASELINE configs[3]: Swin-B MLP stack, per-GPU share of batch
    # 1024 on 8 GPUs = 128 images, 24 layers): tokens/s and fraction of the int8 tensor roof -----
    stack = None
    if rank == 0 and not args.no_stack:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import stack_bench
        stack = stack_bench.run(4, max(3, min(args.steps, 10)), synth.ACT_RELU)
        stack = {k: stack[k] for k in ("workload", "layers", "ms_per_step", "tokens_per_s", "tops", "tensor_frac",
                                       "int8_peak_tops", "stages", "l2")}
        torch.cuda.empty_cache()

    # ---- NEXT-2 row: proj GEMM + fused op #4 (+LN2), one kernel per layer --------
    proj = None
    if rank == 0 and not args.no_stack:
        proj = proj_rows(max(3, min(args.steps, 20)))
    # ---- BASELINE configs[2] / configs[3] as the target states them: a FIXED global batch sharded by
    # whole images over the N ranks (strong scaling; per-GPU T shrinks as N grows), weights broadcast
    # once over NCCL, no collective inside the timed region, max over ranks ------------------------
    sharded = None
    if not args.no_stack:
        sharded = [sharded_stack(cfg, ws, rank, dev, max(3, min(args.steps, 10)), barrier, max_over_ranks)
                   for cfg in (3, 4)]
        torch.cuda.empty_cache()
    # ---- NEXT-3 / NEXT-4 rows: op #1, QKV GEMM + op #2, window-attention core at the
    # Swin-T b64 stage shapes (the attention half of the same blocks) ---------------------------------
    attn_half = None
    if rank == 0 and not args.no_stack:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import attn_bench
        attn_half = attn_bench.run("swin_t", max(5, min(args.steps, 20)))
    # ---- BASELINE configs[0]: one 7x7 window of the Swin-T stage-4 MLP (T = 49), latency ------------
    cfg1 = None
    if rank == 0 and not args.no_stack:
        cfg1 = window_latency(max(10, min(args.steps, 50)))

    # ---- CPU baseline: the oracle as it stands on this host (rank 0, N=1 only) ----------------------
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        rate, tok, t, nth = cpu_oracle_rate(layers_spec(args.batch, synth.ACT_RELU), args.cpu_stride)
        cpu = {"value": rate, "unit": "tokens/s", "cores": nth, "kind": "oracle",
               "sample": f"every {args.cpu_stride}th token of each of the 4 layers ({tok} tokens, {t:.1f} s)",
               "cpu_model": cpu_model(), "per_C": oracle_per_c_table()}

    plans = [l.plan(T) for (_, T, _), l in zip(spec, relu_layers)]
    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": t_ms / args.steps, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "s8", "data": "synthetic",
                "config": {"workload": WORKLOAD, "layers": [{"C": L.C, "H": L.H, "T": T} for (L, T, _) in spec],
                           "act": "relu (GELU-less, b1=None)", "parallelism": f"token-shard weak x{ws}",
                           "l2": "flushed between steps (256 MiB write, untimed)", "plans": plans},
                "roofline": roofline, "cpu_baseline": cpu,
                "e2e": {"value": e2e_val, "unit": "tokens/s", "h2d_bytes_per_step": h2d,
                        "d2h_bytes_per_step": d2h, "steps": e2e_steps, "api": "swin_mlp_int8_run_host_batch",
                        "per_layer_run_host": res_e2e["per_layer"]},
                "gpu_launches": sum(n * P.swin_mlp_int8_launches_per_run(l.handle) for (_, _, n), l in zip(prof, relu_layers)),
                "relu_vs_gelu": relu_gelu,
                "north_star_stack": stack,
                "sharded_fixed_batch": sharded,
                "proj_op4": proj,
                "attention_half": attn_half,
                "config0_window": cfg1,
                "tensor_frac_of_step": roofline["step_frac"],
                "clocks": sampler.result()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.barrier()
        dist.destroy_process_group()


def sharded_stack(config, ws, rank, dev, steps, barrier, max_over_ranks):
    """BASELINE configs[2] (synth config 3: Swin-S MLP stack, batch 256) and configs[3] (config 4:
    Swin-B, batch 1024) with the global batch FIXED and split by whole images over the ws ranks
    (paper_2402_01169_b200.dist.shard_range): rank r runs every layer of the stack on its images'
    tokens.  Weights: rank 0's, broadcast once over NCCL before timing (the only collective; a
    checksum all-gathered afterwards proves every rank holds the same bytes).  Timed: `steps` stack
    passes, L2 flushed before each, CUDA events on the launching stream, job time = max over ranks;
    tokens/s counts the whole batch's layer-tokens.  "scaling": "strong"."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import synth
    from paper_2402_01169_b200 import SwinMlpInt8Layer, swin_mlp_int8_workspace_bytes
    from paper_2402_01169_b200.dist import broadcast_layer, shard_range
    full_batch = {3: 256, 4: 1024}[config]
    lo, hi = shard_range(full_batch, rank, ws)
    stages_full = synth.config_layers(config)
    stages = synth.config_layers(config, batch=hi - lo)
    layers, bufs, wsb, csum = [], [], 128, 0
    for s_i, (C, T, n) in enumerate(stages):
        L0 = synth.make_layer(C, synth.layer_seed(config, s_i, 0))
        a = torch.from_numpy(synth.make_activations(L0, T, synth.layer_seed(config, s_i, 0) + 50 + 7919 * rank)).to(dev)
        bufs.append((a, torch.empty_like(a)))
        for l_i in range(n):
            L = synth.make_layer(C, synth.layer_seed(config, s_i, l_i))
            if ws > 1:
                broadcast_layer(L, dev)
                csum += int(L.w1.to(torch.int64).sum().item()) * 3 + int(L.w2.to(torch.int64).sum().item())
            h = SwinMlpInt8Layer(L, device=dev.index)
            layers.append((h, s_i, l_i, T))
            wsb = max(wsb, swin_mlp_int8_workspace_bytes(h.handle, T))
    work = torch.empty(wsb, dtype=torch.uint8, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream(dev)

    def step():
        for h, s_i, l_i, T in layers:
            a, b = bufs[s_i]
            x, y = (a, b) if l_i % 2 == 0 else (b, a)
            h(x, y=y, workspace=work)

    for _ in range(3):
        step()
    barrier()
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    for k in range(steps):
        flush.fill_(k & 0xff)
        evs[k][0].record(stream)
        step()
        evs[k][1].record(stream)
    torch.cuda.synchronize(dev)
    barrier()
    ms = max_over_ranks(sum(a.elapsed_time(b) for a, b in evs))
    checks_equal = True
    if ws > 1:
        allc = [None] * ws
        dist.all_gather_object(allc, csum)
        checks_equal = len(set(allc)) == 1
    tokens = sum(T * n for (C, T, n) in stages_full)
    ops = sum(16.0 * C * C * T * n for (C, T, n) in stages_full)
    peak = 2.0 * load_peaks()["bf16_burst"]
    t = ms / steps / 1e3
    out = {"config": f"BASELINE configs[{config - 1}]", "workload": {3: "Swin-S MLP stack (24 layers)",
                                                                     4: "Swin-B MLP stack (24 layers)"}[config],
           "global_batch": full_batch, "images_per_gpu": hi - lo, "n_gpus": ws, "scaling": "strong",
           "per_gpu_T": [T for (_, T, _) in stages], "C": [C for (C, _, _) in stages],
           "ms_per_step": ms / steps, "tokens_per_s": tokens / t, "layer_tokens_per_step": tokens,
           "tensor_frac_per_gpu": ops / t / 1e12 / ws / peak,
           "weights": "rank 0's, broadcast once over NCCL before timing" if ws > 1 else "local (1 GPU)",
           "weights_checksum_equal_across_ranks": checks_equal,
           "hot_path_collectives": 0, "l2": "flushed between steps",
           "plans": [h.plan(T)["run_plan"] if not h.plan()["fused"] else "fused" for h, _, l_i, T in layers if l_i == 0]}
    del layers
    return out


def window_latency(steps):
    """BASELINE configs[0]: Swin-T stage-4 MLP (C = 768 -> 3072 -> 768) on
    one 7x7 window, T = 49 tokens, batch 1.  Latency-bound: reported as us per layer, cold (L2
    flushed before each run: the 4.7 MB of weights come from HBM) and hot (back to back), the
    hot time per layer inside a CUDA graph of `steps` layer runs (launch overhead removed), and
    the fraction of the HBM roof for the cold run's algorithmic bytes (weights + 2C per token)."""
    import torch
    import synth
    from paper_2402_01169_b200 import SwinMlpInt8Layer
    peak_gbs = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
    L = synth.make_layer(768, synth.layer_seed(1, 3, 0))
    layer = SwinMlpInt8Layer(L, device=0)
    T = 49
    x = torch.from_numpy(synth.make_activations(L, T, 3)).cuda()
    y = torch.empty_like(x)
    ws = layer.workspace(T)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for _ in range(5):
        layer(x, y=y, workspace=ws)
    torch.cuda.synchronize()

    def run(cold):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            if cold:
                flush.fill_(k & 0xff)
            ev[k][0].record()
            layer(x, y=y, workspace=ws)
            ev[k][1].record()
        torch.cuda.synchronize()
        return sorted(a.elapsed_time(b) * 1e3 for a, b in ev)[steps // 2]

    cold, hot = run(True), run(False)
    try:
        graph_us = graph_time(torch, layer, x, y, ws, steps)
    except Exception as e:   # (reported, never fatal to the bench line)
        graph_us = f"capture failed: {e}"[:200]
    bytes_cold = 2 * 4 * 768 * 768 + 2 * 768 * T
    return {"workload": "configs[0]: Swin-T stage-4 MLP, one 7x7 window (T = 49), batch 1, int8",
            "us_cold_l2": round(cold, 2), "us_hot_l2": round(hot, 2),
            "us_hot_in_cuda_graph": round(graph_us, 2) if isinstance(graph_us, float) else graph_us,
            "hbm_frac_cold": round(bytes_cold / (cold * 1e-6) / 1e9 / peak_gbs, 3),
            "algorithmic_bytes": bytes_cold, "plan": layer.plan(T), "parallelism": "replicas only (DESIGN.md §2.6)"}


def graph_time(torch, layer, x, y, ws, steps):
    """Per-layer time of `steps` layer runs captured in one CUDA graph (no launch overhead)."""
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        layer(x, y=y, workspace=ws)   # (warm the map cache on this stream)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(steps):
                layer(x, y=y, workspace=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    g.replay()
    torch.cuda.synchronize()
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / steps


def proj_rows(steps):
    """Proj GEMM + op #4 (+LN2) (swin_proj_int8_run) at the Swin-T b64 stage shapes and the Swin-B
    b128 stage-3 shape: CUDA events on the launching stream around `steps` back-to-back launches,
    L2 flushed before each; ops = 2*T*C*C per launch (int8 tensor roof)."""
    import torch
    import synth
    from paper_2402_01169_b200 import SwinProjInt8Layer
    peak = 2.0 * json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["bf16_tflops"]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows = []
    for C, T in ((96, 200704), (192, 50176), (384, 12544), (768, 3136), (512, 25088)):
        Pl = synth.make_proj(C, synth.layer_seed(2, 0, 90) + C)
        layer = SwinProjInt8Layer(Pl, device=0)
        a = torch.from_numpy(synth.make_attn_out(Pl, T, 5)).cuda()
        r = torch.from_numpy(synth.make_residual(T, C, 6)).cuda()
        y = torch.empty_like(a)
        z = torch.empty_like(r)
        for _ in range(3):
            layer(a, r, y=y, residual_out=z)
        torch.cuda.synchronize()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        for k in range(steps):
            flush.fill_(k & 0xff)
            ev[k][0].record()
            layer(a, r, y=y, residual_out=z)
            ev[k][1].record()
        torch.cuda.synchronize()
        us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ev)[steps // 2]
        tops = 2.0 * T * C * C / (us * 1e-6) / 1e12
        rows.append({"C": C, "T": T, "us_median": round(us, 2), "tokens_per_s": T / (us * 1e-6),
                     "tops": round(tops, 1), "tensor_frac": round(tops / peak, 3),
                     "hbm_gbs": round((2 * C + 8 * C) * T / (us * 1e-6) / 1e9, 1), "plan": layer.plan()})
        del layer
    return {"what": "swin_proj_int8_run: Proj GEMM + op #4 + LN2 (PAPER.md Fig. 1 lines 63-70, reading R18)",
            "bytes_per_token": "C (a) + 4C (residual) + C (y) + 4C (z)", "rows": rows, "steps": steps}


if __name__ == "__main__":
    main()
