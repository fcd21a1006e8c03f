"""Shared helpers for the test suite (imported as a plain module)."""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def cuda_ready():
    try:
        import torch
        from paper_1903_07525_b200 import _lib
        return torch.cuda.is_available() and _lib.library_available()
    except Exception:
        return False
