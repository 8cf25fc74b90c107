import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA sm_100 device (B200)")
    config.addinivalue_line("markers", "slow: long-running")


def golden(name):
    p = GOLDEN / name
    if p.suffix == ".json":
        return json.loads(p.read_text())
    return np.load(p)


def unhex(xs):
    return np.array([float.fromhex(x) for x in xs], np.float64)


@pytest.fixture(scope="session")
def oracle():
    from oracle.bind import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def ref():
    """The reference library compiled from /root/reference (oracle/_ref).
    Built in the build container by __graft_entry__.build(); shipped prebuilt
    to the GPU box. Tests that need it skip when it is absent."""
    from oracle.bind import REF_SO, Ref
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libpars_ref.so not built")
    r = Ref()
    r.set_threads(1)
    return r


@pytest.fixture(scope="session")
def ctx():
    """CUDA context on device 0. No fallback: a missing extension or device
    is a hard failure for every gpu-marked test."""
    from paper_2510_03243_b200 import Context
    c = Context(0)
    yield c
    c.close()


def extractor_from(desc):
    from paper_2510_03243_b200 import Extractor
    return Extractor.make(dim=desc["dim"], word=tuple(desc["word"]), char=tuple(desc["char"]),
                          norm="l2" if desc["norm"] == 1 else "none",
                          kind="hashed" if desc["kind"] == 0 else "embedding")
