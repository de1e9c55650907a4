"""lm_fill_pcg64 reproduces numpy's default_rng(seed).uniform stream bit for
bit (the SURVEY.md 8(d) operand scheme generated in device memory)."""

import numpy as np
import pytest
import torch

from paper_2502_03000_b200.batch import empty_batch
from paper_2502_03000_b200.datagen import fill_batch_class, fill_seeded, host_batch_instance, host_draws, CHUNK
from paper_2502_03000_b200.matrix import fortran_empty

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(1, 1), (1, 300), (300, 1), (33, 17), (64, 64), (100, 513), (4096, 7)])
@pytest.mark.parametrize("seed", [0, 42, [1000003 * 42 + 505, 64, 3]])
def test_matrix_matches_numpy(shape, seed):
    r, c = shape
    t = fill_seeded(fortran_empty(r, c), seed)
    want = np.random.default_rng(seed).uniform(-1.0, 1.0, (r, c))
    assert np.array_equal(t.cpu().numpy(), want)


def test_skip_row_stream_and_bounds():
    seed = 1234
    t = fill_seeded(fortran_empty(5, 9), seed, skip=1000, row_stream=77, lo=2.0, hi=5.0)
    h = t.cpu().numpy()
    for i in range(5):
        assert np.array_equal(h[i], host_draws(seed, 1000 + 77 * i, 9, 2.0, 5.0))
    # a strided (ld > rows) window of a larger matrix: only the window is written
    big = torch.zeros((40, 20), dtype=torch.float64, device="cuda").t().contiguous().t()
    fill_seeded(big[3:13, 2:8], seed)
    hb = big.cpu().numpy()
    assert np.array_equal(hb[3:13, 2:8], np.random.default_rng(seed).uniform(-1, 1, (10, 6)))
    hb[3:13, 2:8] = 0
    assert not hb.any()


@pytest.mark.parametrize("dtype", [torch.float64, torch.float32])
def test_batch_and_f32_rounding(dtype):
    seed = [7, 8]
    t = fill_seeded(empty_batch(6, 32, 32, dtype), seed)
    want = np.random.default_rng(seed).uniform(-1, 1, (6, 32, 32))
    if dtype == torch.float32:
        want = want.astype(np.float32)
    assert np.array_equal(t.cpu().numpy(), want)


def test_batch_class_chunks_cross_boundaries():
    n = 32
    first, count = CHUNK - 3, 10  # straddles chunks 0 and 1
    t = fill_batch_class(empty_batch(count, n, n), 2, n, first)
    h = t.cpu().numpy()
    for i in range(count):
        assert np.array_equal(h[i], host_batch_instance(2, n, first + i)), i
