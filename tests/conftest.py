import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running CPU test")


@pytest.fixture(scope="session")
def golden():
    import numpy as np
    return np.load(os.path.join(ROOT, "tests", "golden", "reference_golden.npz"))


@pytest.fixture(scope="session")
def port32():
    import numpy as np
    from oracle.pyoracle import Port
    return Port(np.float32)


@pytest.fixture(scope="session")
def port64():
    import numpy as np
    from oracle.pyoracle import Port
    return Port(np.float64)


@pytest.fixture(scope="session")
def ref():
    from oracle.pyoracle import REF_LIB, Ref
    if not os.path.exists(REF_LIB):
        pytest.skip("oracle/_ref not built (reference not available)")
    return Ref()
