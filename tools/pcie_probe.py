"""PCIe probe (dev aid): pinned H2D / D2H bandwidth alone and concurrent, 1 GiB."""
import torch
n = 1 << 28
h_in = torch.empty(n, dtype=torch.int32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.int32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.int32, device="cuda")
d_b = torch.empty(n, dtype=torch.int32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=5):
    ts = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts)
def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
gb = n * 4 / 1e9
h2d = t(lambda: d_a.copy_(h_in, non_blocking=True))
d2h = t(lambda: h_out.copy_(d_b, non_blocking=True))
bo = t(both)
print(f"H2D {gb/h2d*1e3:.1f} GB/s ({h2d:.2f} ms), D2H {gb/d2h*1e3:.1f} GB/s ({d2h:.2f} ms), "
      f"concurrent {bo:.2f} ms = {2*gb/bo*1e3:.1f} GB/s total")
