import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden", "reference_fields.npz")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); run with -m gpu")


@pytest.fixture(scope="session")
def golden():
    return np.load(GOLDEN)


def golden_cases(g):
    """Yield (key, counts, lengths, family, r, i, alg, draws, field) per golden case."""
    keys = sorted({k.rsplit("_", 1)[0] for k in g.files if k.endswith("_field")})
    for key in keys:
        yield (key, tuple(g[key + "_counts"]), tuple(g[key + "_lengths"]), int(g[key + "_family"]),
               g[key + "_r"], g[key + "_i"], int(key.split("_a")[1]), g[key + "_draws"], g[key + "_field"])


def rel_l2(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))
