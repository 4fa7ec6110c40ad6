"""Pinned host<->device copy bandwidth on this box (the e2e leg's transfer ceiling)."""
import torch

d = torch.device("cuda", 0)
for nbytes in (6_220_800, 24_883_200, 268_435_456):
    dev_buf = torch.empty(nbytes, dtype=torch.uint8, device=d)
    host = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
    for name, fn in (("D2H", lambda: host.copy_(dev_buf, non_blocking=True)),
                     ("H2D", lambda: dev_buf.copy_(host, non_blocking=True))):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 20
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / n
        print(f"{name} {nbytes / 1e6:8.1f} MB: {ms * 1e3:8.1f} us  {nbytes / ms / 1e6:6.1f} GB/s")
