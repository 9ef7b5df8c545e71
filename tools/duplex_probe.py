"""PCIe duplex check: pinned H2D alone, D2H alone, and both at once on two
streams (the e2e leg's transfer floor)."""
import torch

MB = 1 << 20
h_in = torch.empty(183 * MB // 4, dtype=torch.float32).pin_memory()
h_out = torch.empty(115 * MB // 4, dtype=torch.float32).pin_memory()
d_in = torch.empty_like(h_in, device="cuda")
d_out = torch.empty_like(h_out, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    for s in (s1, s2):
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)


def both():
    h2d()
    d2h()


for name, fn, mb in (("H2D 183MB", h2d, 183), ("D2H 115MB", d2h, 115), ("both", both, 298)):
    ms = timed(fn)
    print(f"{name:10s}: {ms:6.2f} ms  {mb / 1024 / (ms / 1e3):6.1f} GB/s")
