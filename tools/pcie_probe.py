#!/usr/bin/env python
"""Pinned host<->device copy bandwidth at the e2e transfer sizes."""
import torch
for kb in (8, 128, 512, 1024, 4096, 65536):
    n = kb * 1024
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    st = torch.cuda.Stream()
    res = {}
    for name, fn in (("H2D", lambda: d.copy_(h, non_blocking=True)), ("D2H", lambda: h.copy_(d, non_blocking=True))):
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
        st.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        with torch.cuda.stream(st):
            e0.record()
            for _ in range(20):
                fn()
            e1.record()
        e1.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / 20
        res[name] = (us, n / us / 1e3)
    print(f"{kb:6d} KB: H2D {res['H2D'][0]:8.1f} us {res['H2D'][1]:6.1f} GB/s | D2H {res['D2H'][0]:8.1f} us {res['D2H'][1]:6.1f} GB/s")
