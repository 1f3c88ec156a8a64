"""Summarise the round's ncu evidence into profiles/.

  python tools/ncu_summary.py <round-tag>

Reads gpurun_out/launches_<tag>.csv (the gpu__time_duration launch list of
`bench.py --steps 2 --warmup 1 --pairs 1 --no-cpu`) and gpurun_out/full_stage{0..3}.ncu-rep
(`ncu --set full` of tools/prof_layer.py <stage>: the 2nd run's kernels),
writes profiles/<tag>_launches.csv, profiles/<tag>_ncu_summary.md and
profiles/ncu_traffic.json (DRAM bytes per launch, keyed like bench.py's kernels).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import synth  # noqa: E402

tag = sys.argv[1] if len(sys.argv) > 1 else "r1"


def fused_stage(L):
    """The one-kernel plan covers C <= 256 with H % 128 == 0 (swin_mlp_int8.cu make_fused)."""
    return L.C <= 256 and L.H % 128 == 0


def step_kernel_names():
    names = []
    for L, T, _ in synth.swin_t_batch64_layers():
        if fused_stage(L):
            names.append(f"fused_mlp[C={L.C},T={T}]")
        else:
            names += [f"fc1_relu_q[C={L.C},T={T}]", f"fc2_ln_q[C={L.C},T={T}]"]
    return names
out = os.path.join(ROOT, "profiles")
os.makedirs(out, exist_ok=True)
lines = []

# ---- launch list
src = os.path.join(ROOT, "gpurun_out", f"launches_{tag}.csv")
if os.path.exists(src):
    shutil.copy(src, os.path.join(out, f"{tag}_launches.csv"))
    txt = open(src).read()
    body = txt[txt.index('"ID"'):] if '"ID"' in txt else txt
    rows = list(csv.DictReader(io.StringIO(body)))
    per, ours_seq = {}, []
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        v = float(r["Metric Value"].replace(",", ""))
        unit = r.get("Metric Unit", "")
        us = v / 1000.0 if unit == "ns" else v if unit == "us" else v * 1000.0 if unit == "ms" else v
        key = "fused_mlp_kernel" if "fused_mlp_kernel" in name else \
            "mlp_gemm_kernel" if "mlp_gemm_kernel" in name else name[:60]
        per.setdefault(key, []).append(us)
        if key in ("fused_mlp_kernel", "mlp_gemm_kernel"):
            ours_seq.append(us)
    lines.append(f"## Launch list (`ncu --metrics gpu__time_duration.sum --clock-control none`, {tag})\n")
    lines.append("Cold-cache, serialised per-launch times: compare shares, not absolutes.\n")
    lines.append("| kernel | launches | total us | mean us |")
    lines.append("|---|---|---|---|")
    tot = sum(sum(v) for v in per.values())
    for k, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{k}` | {len(v)} | {sum(v):.1f} | {sum(v)/len(v):.2f} |")
    names = step_kernel_names()
    n = len(names)
    if len(ours_seq) >= 2 * n:
        lines.append(f"\nOur kernels: {len(ours_seq)} launches, {sum(ours_seq):.1f} us of {tot:.1f} us listed "
                     f"({sum(ours_seq)/tot:.1%}; the rest is the L2-flush fill, copies and torch setup).\n")
        step = ours_seq[n:2 * n]      # the second step (warm)
        lines.append(f"Per-launch share of one step (launches {n + 1}-{2 * n}):\n")
        lines.append("| launch | us | share |")
        lines.append("|---|---|---|")
        for nm, us in zip(names, step):
            lines.append(f"| {nm} | {us:.2f} | {us/sum(step):.1%} |")

# ---- full captures
METRICS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
           "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
           "sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active",
           "smsp__issue_active.avg.pct_of_peak_sustained_active",
           "lts__t_bytes.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
           "lts__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
           "launch__grid_size", "launch__cluster_dim_x"]
traffic = {}
lines.append("\n## `ncu --set full` captures (tools/prof_layer.py <stage>, 2nd run; one launch each)\n")
lines.append("| kernel | us | DRAM read MB | DRAM write MB | L2 bytes MB (32 x lts__t_sectors) | tensor(imma) % active | issue % | L2 % | regs | grid | cluster |")
lines.append("|---|---|---|---|---|---|---|---|---|---|---|")
specs = synth.swin_t_batch64_layers()
for st in range(4):
    rep = os.path.join(ROOT, "gpurun_out", f"full_stage{st}.ncu-rep")
    raw_csv = os.path.join(ROOT, "gpurun_out", f"full_stage{st}_raw.csv")   # exported on the box
    if os.path.exists(raw_csv):
        raw = open(raw_csv).read()
        shutil.copy(raw_csv, os.path.join(out, f"{tag}_full_stage{st}_raw.csv"))
        det = raw_csv.replace("_raw.csv", "_details.csv")
        if os.path.exists(det):
            shutil.copy(det, os.path.join(out, f"{tag}_full_stage{st}_details.csv"))
        if os.path.exists(rep):
            shutil.copy(rep, os.path.join(out, f"{tag}_full_stage{st}.ncu-rep"))
    elif os.path.exists(rep):
        shutil.copy(rep, os.path.join(out, f"{tag}_full_stage{st}.ncu-rep"))
        raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    else:
        continue
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units, data = rr[0], rr[1], rr[2:]
    L, T, _ = specs[st]
    for j, row in enumerate(data):
        d = {h: row[i] for i, h in enumerate(hdr)}
        u = {h: units[i] for i, h in enumerate(hdr)}

        def val(m, scale_to=None):
            v = float(d.get(m, "nan").replace(",", "") or "nan")
            un = u.get(m, "")
            if scale_to == "MB":
                f = {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(un, 1)
                return v * f
            if scale_to == "us":
                f = {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(un, 1)
                return v * f
            return v
        name = f"fused_mlp[C={L.C},T={T}]" if fused_stage(L) else \
            f"{'fc1_relu_q' if j == 0 else 'fc2_ln_q'}[C={L.C},T={T}]"
        rd, wr = val("dram__bytes_read.sum", "MB"), val("dram__bytes_write.sum", "MB")
        traffic[name] = (rd + wr) * 1e6
        lines.append(f"| {name} | {val('gpu__time_duration.sum', 'us'):.1f} | {rd:.1f} | {wr:.1f} | "
                     f"{val('lts__t_sectors.sum') * 32e-6:.1f} | "
                     f"{val('sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{val('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{val('lts__throughput.avg.pct_of_peak_sustained_elapsed'):.1f} | "
                     f"{d.get('launch__registers_per_thread', '')} | {d.get('launch__grid_size', '')} | "
                     f"{d.get('launch__cluster_dim_x', '')} |")
# extra captures: the north-star stage (Swin-B b128 stage 3, C = 512) and the attention half
extra = {"swinb3": ("Swin-B b128 stage 3 layer (C=512, T=25088)", ["fc1_relu_q", "fc2_ln_q"]),
         "attn0": ("attention half, Swin-T b64 stage 0 (C=96, T=200704)", ["op1", "qkv_op2", "attn_core"]),
         "config0": ("configs[0]: one 7x7 window (C=768, T=49), the one-launch plan", ["small_mlp (one launch)"])}
for key, (what, names) in extra.items():
    raw_csv = os.path.join(ROOT, "gpurun_out", f"full_stage{key}_raw.csv")
    if not os.path.exists(raw_csv):
        continue
    shutil.copy(raw_csv, os.path.join(out, f"{tag}_full_{key}_raw.csv"))
    det = raw_csv.replace("_raw.csv", "_details.csv")
    if os.path.exists(det):
        shutil.copy(det, os.path.join(out, f"{tag}_full_{key}_details.csv"))
    rr = list(csv.reader(open(raw_csv)))
    hdr, units, data = rr[0], rr[1], rr[2:]
    lines.append(f"\n### {what}\n")
    lines.append("| kernel | us | DRAM read MB | DRAM write MB | tensor(imma) % | issue % | eligible warps/sched | regs | grid |")
    lines.append("|---|---|---|---|---|---|---|---|---|")
    for jj, row in enumerate(data):
        d = {h: row[i] for i, h in enumerate(hdr)}
        u = {h: units[i] for i, h in enumerate(hdr)}

        def v2(m, scale_to=None):
            try:
                v = float(d.get(m, "nan").replace(",", "") or "nan")
            except ValueError:
                return float("nan")
            un = u.get(m, "")
            if scale_to == "MB":
                return v * {"byte": 1e-6, "Kbyte": 1e-3, "Mbyte": 1, "Gbyte": 1e3}.get(un, 1)
            if scale_to == "us":
                return v * {"nsecond": 1e-3, "usecond": 1, "msecond": 1e3}.get(un, 1)
            return v
        nm = names[jj] if jj < len(names) else d.get("Kernel Name", "")[:40]
        lines.append(f"| {nm} | {v2('gpu__time_duration.sum', 'us'):.1f} | {v2('dram__bytes_read.sum', 'MB'):.1f} | "
                     f"{v2('dram__bytes_write.sum', 'MB'):.1f} | "
                     f"{v2('sm__pipe_tensor_subpipe_imma_cycles_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{v2('smsp__issue_active.avg.pct_of_peak_sustained_active'):.1f} | "
                     f"{v2('smsp__warps_eligible.avg.per_cycle_active'):.2f} | "
                     f"{d.get('launch__registers_per_thread', '')} | {d.get('launch__grid_size', '')} |")
json.dump(traffic, open(os.path.join(out, "ncu_traffic.json"), "w"), indent=1)
open(os.path.join(out, f"{tag}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
print("\n".join(lines))
