import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _limit_blas():
    """OpenBLAS with one thread per logical core hits shape-dependent threading pathologies
    (100x slowdowns on skinny products); half the cores, at most 8, is reliably fast."""
    try:
        from threadpoolctl import threadpool_limits
        n = max(1, min(8, len(os.sched_getaffinity(0)) // 2))
        return threadpool_limits(n, user_api="blas")
    except Exception:
        return None


_BLAS_LIMIT = _limit_blas()


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU; parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: longer CPU oracle runs")


def pytest_collection_modifyitems(config, items):
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:
        has_gpu = False
    if has_gpu:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
