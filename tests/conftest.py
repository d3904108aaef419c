"""Shared fixtures.  ``-m gpu`` tests need a B200 and call the product
through its C ABI; everything else runs on CPU (oracle, host logic, ABI
symbol checks)."""
from __future__ import annotations

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

REFERENCE_SRC = "/root/reference/pkg/src"

#: Codes used throughout (GbSpec arguments).
TOY = (3, (0, 1), (0, 2))                                   # [[6,2]] twin columns
SMALL = (5, (0, 1), (0, 2))                                  # [[10,2]]
GB126 = (63, (0, 1, 14, 16, 22), (0, 3, 13, 20, 42))         # [[126,28]]
GB254 = (127, (0, 15, 20, 28, 66), (0, 58, 59, 100, 121))    # [[254,28]] BASELINE
GB1022 = (511, (0, 5, 200, 397, 418), (0, 81, 284, 347, 418))  # l=511 w=5


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "reference: needs /root/reference importable (this container only)")
    config.addinivalue_line("markers", "slow: long-running")


def have_reference() -> bool:
    return os.path.isdir(REFERENCE_SRC)


@pytest.fixture(scope="session")
def reference():
    """The reference package, imported in place (CPU container only)."""
    if not have_reference():
        pytest.skip("reference not present (GPU box)")
    if REFERENCE_SRC not in sys.path:
        sys.path.insert(0, REFERENCE_SRC)
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    sys.dont_write_bytecode = True
    import qsagms  # noqa: F401
    return qsagms


@pytest.fixture(scope="session")
def oracle():
    from oracle import oracle as O
    O.lib()
    return O


def make_tree_rows(rng, n_target):
    """Random cycle-free check matrix (reference tests/conftest.py:48-68
    restated): each new check joins one existing qubit and 1-2 fresh ones."""
    rows, n = [], 1
    while n < n_target:
        anchor = int(rng.integers(0, n))
        fresh = min(int(rng.integers(1, 3)), n_target - n)
        if fresh == 0:
            break
        members = [anchor] + list(range(n, n + fresh))
        n += fresh
        rows.append(sorted((j, int(rng.integers(1, 4))) for j in members))
    return n, rows
