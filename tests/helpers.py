"""Shared test helpers (paths, reference-availability gate)."""
import os

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def have_ref() -> bool:
    return os.path.exists(os.path.join(ROOT, "oracle", "_ref", "liblatecache_ref.so"))


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:  # noqa: BLE001
        return False


requires_ref = pytest.mark.skipif(not have_ref(), reason="oracle/_ref (compiled reference) not built")
