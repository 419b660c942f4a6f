import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: long-running case")


def _ensure_built():
    # Build the oracle (C restatement; the reference .so is prebuilt here and
    # travels with the snapshot) and the product library if missing.
    orc = os.path.join(ROOT, "oracle", "build", "liboracle.so")
    if not os.path.exists(orc):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "oracle"), "oracle"], check=True)
    lib = os.path.join(ROOT, "paper_2603_10353_b200", "lib", "libshplb.so")
    if not os.path.exists(lib):
        subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "paper_2603_10353_b200", "csrc"),
                        "-j8"], check=True)


_ensure_built()


@pytest.fixture(scope="session")
def cuda_ctx():
    import torch

    import paper_2603_10353_b200 as P
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    ctx = P.Context(0)
    yield ctx
    ctx.close()
