"""Host<->device copy bandwidth of this box (pinned memory): H2D alone, D2H alone and both at once
on two streams -- the ceiling of bench.py's e2e line (PCIe-bound: ~26.6 GB D2H per C3 step)."""
import json
import torch

GB = 1 << 30
n = 2 * GB // 8
h_src = torch.empty(n, dtype=torch.float64, pin_memory=True)
h_dst = torch.empty(n, dtype=torch.float64, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float64, device="cuda")
d_b = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / 1e3 / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)


def d2h():
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s2)


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)


b = n * 8
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_gbs": b / t1 / 1e9, "d2h_gbs": b / t2 / 1e9, "bidir_h2d_plus_d2h_gbs": 2 * b / t3 / 1e9,
                  "bytes_per_copy": b}))
