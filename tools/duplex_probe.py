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


# the e2e leg's actual copy mix: per-array H2D copies (hoisted copyins of
# yolov2-tiny, MB) on one stream and per-array D2H copies on another
sizes_in = [17.8, 0.0001, 10.6, 0.002, 2.6, 23.8, 0.0001, 5.3, 0.02, 1.3, 11.9, 0.0003, 2.6, 0.07,
            0.7, 5.9, 0.0005, 1.3, 0.3, 0.3, 3.0, 0.001, 0.7, 1.1, 0.2, 1.5, 0.002, 0.3, 4.5, 0.3,
            3.0, 0.004, 0.7, 18.0, 5.9, 0.002, 0.3, 18.0, 0.002, 0.3, 0.8] + [2.0] * 16
sizes_out = [17.8, 10.6, 2.6, 2.6, 23.8, 5.3, 1.3, 1.3, 11.9, 2.6, 0.7, 0.7, 5.9, 1.3, 0.3, 0.3, 3.0,
             0.7, 0.2, 0.2, 1.5, 0.3, 0.3, 0.3, 3.0, 0.7, 5.9, 0.3, 0.3, 0.3]
def views(total, sizes):
    out, off = [], 0
    for mb in sizes:
        n = max(1, int(mb * MB / 4))
        out.append((off, n))
        off += n
    return out
vin, vout = views(h_in.numel(), sizes_in), views(h_out.numel(), sizes_out)


def h2d_many():
    with torch.cuda.stream(s1):
        for off, n in vin:
            d_in[off:off + n].copy_(h_in[off:off + n], non_blocking=True)


def d2h_many():
    with torch.cuda.stream(s2):
        for off, n in vout:
            h_out[off:off + n].copy_(d_out[off:off + n], non_blocking=True)


def both_many():
    h2d_many()
    d2h_many()


for name, fn in (("H2D x57", h2d_many), ("D2H x30", d2h_many), ("both many", both_many)):
    print(f"{name:10s}: {timed(fn):6.2f} ms")


def mix_a():
    h2d_many()
    d2h()


def mix_b():
    h2d()
    d2h_many()


for name, fn in (("H2D many + D2H one", mix_a), ("H2D one + D2H many", mix_b)):
    print(f"{name:20s}: {timed(fn):6.2f} ms")


chunks = views(h_in.numel(), [sum(sizes_in) / 8] * 8)


def h2d_8():
    with torch.cuda.stream(s1):
        for off, n in chunks:
            d_in[off:off + n].copy_(h_in[off:off + n], non_blocking=True)


def mix_c():
    h2d_8()
    d2h_many()


print(f"{'H2D x8 + D2H many':20s}: {timed(mix_c):6.2f} ms")
