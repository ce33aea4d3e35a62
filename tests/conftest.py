import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
GOLDEN = Path(__file__).resolve().parent / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built native library")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz") as z:
        return {k: z[k] for k in z.files}


@pytest.fixture(scope="session")
def arm7():
    from paper_2104_13542_b200.kinematics import load_chain

    return load_chain("arm7.chain")


@pytest.fixture(scope="session")
def planar2():
    from paper_2104_13542_b200.kinematics import load_chain

    return load_chain("planar2.chain")


@pytest.fixture(scope="session")
def slider1():
    from paper_2104_13542_b200.kinematics import load_chain

    return load_chain("slider1.chain")


@pytest.fixture
def rng():
    return np.random.default_rng(1234)


@pytest.fixture(scope="session")
def surrogate_state():
    from paper_2104_13542_b200.surrogate import ARM7_SURROGATE

    with np.load(ARM7_SURROGATE) as z:
        return {k: z[k] for k in z.files if k.startswith(("W", "b"))}


def random_q(chain, rng, n=1, margin=0.05):
    lo, hi = chain.joint_limits[:, 0], chain.joint_limits[:, 1]
    span = hi - lo
    q = rng.uniform(lo + margin * span, hi - margin * span, size=(n, chain.dof))
    return q[0] if n == 1 else q
