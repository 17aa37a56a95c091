"""Shared fixtures. `-m gpu` tests need a B200 and libtmd_gpu.so; everything
else runs on the CPU (the oracle, host logic, ABI symbol checks)."""
from __future__ import annotations

import os
import sys
from pathlib import Path

import pytest

# the native slab loop falls back to the message halo when a rank cannot map a
# peer's buffers; under test that is an error, so the fused path cannot
# silently degrade (tmd_slab_nccl.cuh, nccl_publish_ghosts)
os.environ.setdefault("TMD_HALO_STRICT", "1")

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libtmd_gpu.so")
    config.addinivalue_line("markers", "slow: long-running (large N or many steps)")


@pytest.fixture(scope="session")
def ref():
    """The reference engine built from /root/reference (oracle/_ref)."""
    from oracle import ref as R
    if not R.available():
        try:
            R.build()
        except Exception as e:  # pragma: no cover
            pytest.skip(f"reference oracle not buildable here: {e}")
    return R
