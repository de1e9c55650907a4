"""Pinned host <-> device copy bandwidth on this box: H2D alone, D2H alone,
and both directions at once on two streams (the e2e ceiling)."""
import time

import torch


def main():
    n = 256 << 20  # bytes per direction
    h_in = torch.empty(n, dtype=torch.uint8).pin_memory()
    h_out = torch.empty(n, dtype=torch.uint8).pin_memory()
    d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
    d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()

    def bench(fn, reps=5):
        fn()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t0) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)

    def both():
        h2d()
        d2h()

    for name, fn, nbytes in (("H2D", h2d, n), ("D2H", d2h, n), ("H2D+D2H", both, 2 * n)):
        t = bench(fn)
        print(f"{name:8s} {nbytes / t / 1e9:7.1f} GB/s  ({t * 1e3:.2f} ms for {nbytes >> 20} MiB)")


if __name__ == "__main__":
    main()
