import json
import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = json.loads((ROOT / "tests" / "golden" / "golden.json").read_text())


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests proper")
    config.addinivalue_line("markers", "slow: long-running CPU oracle checks")


@pytest.fixture(scope="session")
def golden():
    return GOLDEN


def u53(seed, shape):
    return np.random.default_rng(seed).integers(0, 1 << 53, shape, dtype=np.uint64)


def digest(a):
    import hashlib
    a = np.ascontiguousarray(np.asarray(a))
    if a.dtype.kind in "iu":
        a = a.astype("<u8") if a.dtype.kind == "u" else a.astype("<i8")
    return hashlib.sha256(a.tobytes()).hexdigest()


def has_cuda():
    if os.environ.get("SFHR_FORCE_NO_GPU"):
        return False
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
