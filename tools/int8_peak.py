"""Measure the dense INT8 tensor-core peak of this B200 with torch._int_mm (cuBLASLt).

MEASURED_PEAKS.json carries HBM and bf16 numbers only; the INT8 roofline
denominator is measured here the same way (8192^3, best of 10 = burst,
back-to-back for 4 s = sustained) and written to profiles/int8_peak.json.
"""
import json, os, subprocess, sys, time
import torch


def main():
    dev = torch.device("cuda:0")
    n = 8192
    a = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev)
    b = torch.randint(-128, 127, (n, n), dtype=torch.int8, device=dev).t()  # column-major B
    for _ in range(3):
        torch._int_mm(a, b)
    torch.cuda.synchronize()
    ops = 2.0 * n ** 3
    best = 1e9
    for _ in range(10):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(); torch._int_mm(a, b); e.record(); torch.cuda.synchronize()
        best = min(best, s.elapsed_time(e) / 1e3)
    burst = ops / best / 1e12
    # sustained: back to back for ~4 s
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active",
                            "--format=csv,noheader,nounits", "-lms", "200"], stdout=subprocess.PIPE, text=True)
    iters = max(1, int(4.0 / best))
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        torch._int_mm(a, b)
    e.record(); torch.cuda.synchronize()
    smi.terminate(); out = smi.communicate()[0]
    sustained = ops * iters / (s.elapsed_time(e) / 1e3) / 1e12
    clocks = [l.split(",") for l in out.strip().splitlines() if l.strip()]
    res = {"int8_tops_burst": burst, "int8_tops_sustained": sustained, "n": n,
           "how": "torch._int_mm int8 8192^3 (2*N^3 ops): best of 10 (burst), back to back ~4 s (sustained)",
           "gpu": torch.cuda.get_device_name(0), "nproc": os.cpu_count(),
           "clock_samples": clocks[-10:]}
    print(json.dumps(res))
    os.makedirs("gpurun_out", exist_ok=True)
    with open("gpurun_out/int8_peak.json", "w") as f:
        json.dump(res, f, indent=1)


if __name__ == "__main__":
    main()
