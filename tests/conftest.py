"""Shared pytest configuration.

Markers
  gpu  -- needs a CUDA device (B200) and the built C-ABI library; the
          driver runs these on the GPU box with ``-m gpu``.  Everything
          unmarked runs on the CPU-only build container.
"""

import os
import pathlib
import sys

ROOT = pathlib.Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLDEN = ROOT / "tests" / "golden"
if str(GOLDEN) not in sys.path:
    sys.path.insert(0, str(GOLDEN))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running (full BASELINE sizes)")
