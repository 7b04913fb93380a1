"""PCIe H2D / D2H / concurrent bandwidth with pinned buffers (diagnostic)."""
import torch

n = 134217728 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


t_h2d = timeit(lambda: d.copy_(h, non_blocking=True))
t_d2h = timeit(lambda: h2.copy_(d2, non_blocking=True))
t_both = timeit(both)
gb = n * 8 / 1e9
print(f"H2D {t_h2d:.3f} ms ({gb / t_h2d * 1e3:.1f} GB/s)  D2H {t_d2h:.3f} ms ({gb / t_d2h * 1e3:.1f} GB/s)  "
      f"concurrent {t_both:.3f} ms")
