import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built librunlab_gpu.so")


@pytest.fixture(scope="session")
def labeler():
    from paper_2006_09299_b200 import Labeler
    lab = Labeler(0)
    yield lab
    lab.close()
