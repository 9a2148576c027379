"""Pinned host <-> device copy bandwidth: each direction alone and both at once (2 GB each)."""
import torch

n = 2 * 1024**3 // 4
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    fn()
    torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / 1000.0


for _ in range(2):
    t_in = timed(lambda: d_a.copy_(h_in, non_blocking=True))
    t_out = timed(lambda: h_out.copy_(d_b, non_blocking=True))

    def both():
        with torch.cuda.stream(s1):
            d_a.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_b, non_blocking=True)
    t_both = timed(both)
gb = n * 4 / 1e9
print(f"H2D {gb / t_in:.1f} GB/s, D2H {gb / t_out:.1f} GB/s, both at once {2 * gb / t_both:.1f} GB/s aggregate")
