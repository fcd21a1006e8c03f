"""PCIe ceiling for the e2e number: pinned H2D alone, D2H alone, both at once."""
import time
import torch

dev = torch.device("cuda", 0)
n = 256 * 1024 * 1024          # 1 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
d_a = torch.empty(n, dtype=torch.float32, device=dev)
d_b = torch.empty(n, dtype=torch.float32, device=dev)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


gb = n * 4 / 1e9
t = timed(h2d)
print("H2D alone  %.1f GB/s" % (gb / t))
t = timed(d2h)
print("D2H alone  %.1f GB/s" % (gb / t))
t = timed(lambda: (h2d(), d2h()))
print("both       %.1f GB/s each way (%.1f ms for %.2f GB each)" % (gb / t, t * 1e3, gb))
