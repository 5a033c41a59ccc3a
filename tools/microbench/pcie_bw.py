"""Pinned host<->device copy bandwidth on this box: H2D alone, D2H alone, and both at once on two streams
(the e2e leg of bench.py moves 4 input tensors in and 4 results out per step). Prints one JSON line."""
import json

import torch

MB = 200 << 20  # one step's inputs at 32k (4 x 50 MB)
h = torch.empty(MB, dtype=torch.uint8).pin_memory()
h2 = torch.empty(MB, dtype=torch.uint8).pin_memory()
d = torch.empty(MB, dtype=torch.uint8, device="cuda")
d2 = torch.empty(MB, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
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


def h2d():
    d.copy_(h, non_blocking=True)


def d2h():
    h2.copy_(d2, non_blocking=True)


def both():
    main = torch.cuda.current_stream()
    s1.wait_stream(main)
    s2.wait_stream(main)
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    main.wait_stream(s1)
    main.wait_stream(s2)


t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
gb = MB / 1e9
print(json.dumps({"bytes_each": MB, "h2d_GBps": gb / (t1 * 1e-3), "d2h_GBps": gb / (t2 * 1e-3),
                  "both_ms": t3, "both_each_GBps": gb / (t3 * 1e-3), "both_total_GBps": 2 * gb / (t3 * 1e-3)}))
