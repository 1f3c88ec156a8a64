"""PCIe copy probe: H2D, D2H and both concurrently (pinned host buffers)."""
import torch
n = 19 << 20
h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def timeit(fn, reps=20):
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    b.record(); b.synchronize()
    return a.elapsed_time(b) / reps
h2d = timeit(lambda: d_in.copy_(h_in, non_blocking=True))
d2h = timeit(lambda: h_out.copy_(d_out, non_blocking=True))
def both():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
bo = timeit(both)
print(f"H2D {n/h2d/1e6:.1f} GB/s  D2H {n/d2h/1e6:.1f} GB/s  both: {2*n/bo/1e6:.1f} GB/s combined ({bo:.3f} ms vs {h2d+d2h:.3f} serial)")
