import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu)")
    config.addinivalue_line("markers", "slow: long-running")


def golden_names():
    return sorted(p.stem[len("field_"):] for p in GOLDEN.glob("field_*.npz"))


def load_golden(name):
    z = np.load(GOLDEN / f"field_{name}.npz", allow_pickle=False)
    return {k: z[k] for k in z.files}


class Cfg:
    """Plain settings object accepted by the oracle driver."""
    def __init__(self, g):
        self.predictor = str(g["predictor"])
        for k in ("bx", "by", "stride", "radius", "n_max"):
            setattr(self, k, int(g[k]))
        for k in ("lam", "theta", "d_max"):
            setattr(self, k, float(g[k]))


@pytest.fixture(scope="session")
def oracle_mod():
    from oracle import cpu_oracle
    cpu_oracle.lib()
    return cpu_oracle
