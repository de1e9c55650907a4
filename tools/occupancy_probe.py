"""Resident CTAs per SM of the library's persistent kernels (the grid they
launch with / 148), read from an ncu-free run: prints each batched kernel's
launch grid via the launch counter order is not needed -- it simply runs one
small batch per kernel under torch.profiler and lists kernel grids."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2502_03000_b200.batch import atb_schur_trace  # noqa: E402


def main():
    for dt in (torch.float64, torch.float32):
        for n in (32, 64, 128):
            ops = [torch.rand((4096, n, n), dtype=dt, device="cuda").transpose(1, 2) for _ in range(4)]
            with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA], record_shapes=False) as prof:
                atb_schur_trace(*ops)
                torch.cuda.synchronize()
            for e in prof.events():
                if "atb_schur" in e.name:
                    print(dt, n, e.name[:60])


if __name__ == "__main__":
    main()
