"""Bandwidth calibration for small (L2-sized) transfers: torch copy / reduction of
one q_proj activation (2048 x 4096 BF16) with rotating buffers, CUDA events."""
import torch

def timeit(fn, reps=50):
    for _ in range(5):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(reps):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3

n = 2048 * 4096
for nb in (1, 16):
    xs = [torch.randn(n, device="cuda", dtype=torch.float32).to(torch.bfloat16) for _ in range(nb)]
    ys = [torch.empty_like(x) for x in xs]
    acc1 = torch.empty((), device="cuda", dtype=torch.float32)
    us = timeit(lambda i: ys[i % nb].copy_(xs[i % nb]))
    print(f"copy   {nb:2d} bufs: {us:7.2f} us  {2 * 2 * n / us / 1e3:7.0f} GB/s (r+w)")
    us = timeit(lambda i: torch.sum(xs[i % nb], dim=(0,), dtype=torch.float32, out=acc1))
    print(f"sum    {nb:2d} bufs: {us:7.2f} us  {2 * n / us / 1e3:7.0f} GB/s (read)")
    big = torch.empty(8 * n, device="cuda", dtype=torch.bfloat16)
    us = timeit(lambda i: big.zero_())
    print(f"memset 8x       : {us:7.2f} us  {2 * 8 * n / us / 1e3:7.0f} GB/s (write)")
