"""Whole-plan CUDA-graph capture: replays equal eager evaluation bitwise,
and read the leaves at replay time."""

import numpy as np
import pytest
import torch

import paper_2502_03000_b200 as lm

pytestmark = pytest.mark.gpu


def _m(rng, r, c):
    return lm.DenseMatrix(np.asfortranarray(rng.uniform(-1, 1, (r, c))))


def test_capture_fused_program_replays_bitwise_and_tracks_inputs():
    rng = np.random.default_rng(3)
    A, B, C = _m(rng, 300, 200), _m(rng, 300, 200), _m(rng, 300, 200)
    expr = 2 * A + B % C - A / (1 + abs(B))
    g = lm.capture(expr)
    eager = lm.evaluate(expr).data.clone()
    assert torch.equal(g().data, eager)
    # new inputs written in place: the replay sees them
    A.data.copy_(torch.from_numpy(np.asfortranarray(rng.uniform(-1, 1, (300, 200)))).cuda())
    eager2 = lm.evaluate(expr).data.clone()
    assert not torch.equal(eager, eager2)
    assert torch.equal(g().data, eager2)


def test_capture_chain_and_trace():
    rng = np.random.default_rng(4)
    A, B, C, v = _m(rng, 256, 256), _m(rng, 256, 256), _m(rng, 256, 256), _m(rng, 256, 1)
    chain = A * B * C * v
    g = lm.capture(chain)
    assert torch.equal(g().data, lm.evaluate(chain).data)
    t = lm.trace(A * B)
    gt = lm.capture(t)
    assert gt() == lm.evaluate(t)
    gt.replay()  # no host sync
    torch.cuda.synchronize()
    assert float(gt.result.data[0, 0].item()) == lm.evaluate(t)
