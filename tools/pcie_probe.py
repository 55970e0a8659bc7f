"""Host<->device copy rates on the box: one 48 MB page-locked buffer copied
as one cudaMemcpyAsync, as two halves on one stream, and as two halves on
two streams (copy engines in parallel?), each direction."""
import time

import torch

n = 6 * 1024 * 1024  # doubles: 48 MB
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, reps=20):
    fn()
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - w0) / reps


half = n // 2
for name, src, dst in (("h2d", h, d), ("d2h", d, h)):
    one = t(lambda: dst.copy_(src, non_blocking=True))

    def two_one_stream():
        dst[:half].copy_(src[:half], non_blocking=True)
        dst[half:].copy_(src[half:], non_blocking=True)

    def two_streams():
        with torch.cuda.stream(s1):
            dst[:half].copy_(src[:half], non_blocking=True)
        with torch.cuda.stream(s2):
            dst[half:].copy_(src[half:], non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)
    a = t(two_one_stream)
    b = t(two_streams)
    gb = 8 * n / 1e9
    print(f"{name}: one copy {gb / one:.1f} GB/s, two halves one stream "
          f"{gb / a:.1f} GB/s, two streams {gb / b:.1f} GB/s")
# both directions at once
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2 = h  # noqa
    torch.cuda.synchronize()
