"""Write bandwidth probe: torch fill / copy of a 1.13 GB buffer, timed with CUDA events."""
import torch
n = 40 * 100 * 266 * 266
a = torch.empty(n, device="cuda")
b = torch.empty(n, device="cuda")
for name, fn in [("fill", lambda: a.fill_(0.0)), ("fill1", lambda: a.fill_(1.0)), ("copy", lambda: b.copy_(a)),
                 ("sum", lambda: a.sum())]:
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        fn()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    by = 4 * n * (2 if name == "copy" else 1)
    print(f"{name}: {ms*1e3:.1f} us  {by/ms/1e6:.0f} GB/s")
