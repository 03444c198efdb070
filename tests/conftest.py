import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str):
    return np.load(GOLDEN / name, allow_pickle=False)


def golden_ham(m: int, seed: int):
    z = golden(f"ham_m{m}_s{seed}.npz")
    return np.asfortranarray(z["a"]), np.asfortranarray(z["b"])


def rebuild_c1():
    """The BASELINE configs[0] instance (generate(m=500, seed=0)), rebuilt on
    the host from the bit-exact rng streams plus the two construction scalars
    recorded from the reference (generate.py:63-74)."""
    from oracle import bse_oracle as o

    g = golden("c1_m500_s0.npz")
    m = 500
    cm = o.gauss_c_matrix(o.child_seed(0, 0), m, m)
    a = cm @ cm.conj().T + np.eye(m)
    a = (a + a.conj().T) / 2.0
    d = o.gauss_c_matrix(o.child_seed(0, 1), m, m)
    b = (0.5 * float(g["lambda_min_a"]) / float(g["b0_norm"])) * ((d + d.T) / 2.0)
    return np.asfortranarray(a), np.asfortranarray(b), g


@pytest.fixture(scope="session")
def c1_instance():
    return rebuild_c1()
