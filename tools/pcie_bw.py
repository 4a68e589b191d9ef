"""Pinned host<->device copy bandwidth on this box (the e2e ceiling)."""
import torch

n = 671088640 // 8
h = torch.empty(n, dtype=torch.float64).pin_memory()
h2 = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
d2 = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timeit(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


gb = n * 8 / 1e9
t = timeit(lambda: d.copy_(h, non_blocking=True))
print(f"H2D {gb / t * 1e3:.1f} GB/s")
t = timeit(lambda: h2.copy_(d2, non_blocking=True))
print(f"D2H {gb / t * 1e3:.1f} GB/s")
t = timeit(both)
print(f"H2D+D2H concurrent {2 * gb / t * 1e3:.1f} GB/s total, {t:.2f} ms for 2 x {gb:.3f} GB")
