import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def _ensure_built():
    """Build the in-tree native pieces if a fresh checkout lacks them (no-op
    when up to date); same entry the driver uses."""
    import __graft_entry__

    __graft_entry__.build()


def pytest_configure(config):
    _ensure_built()
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); parity tests through the C-ABI")
    config.addinivalue_line("markers", "slow: full-size BASELINE configurations")


def _cuda_ok() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if _cuda_ok():
        return
    skip = pytest.mark.skip(reason="no CUDA device in this container")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def orc():
    import oracle

    return oracle.orc()


@pytest.fixture(scope="session")
def ref():
    import oracle

    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built (needs /root/reference at build time)")
    return oracle.ref()


@pytest.fixture(scope="session")
def corpus(ref):
    """The reference test corpus (proj/tests/support.hpp:86-119), 500 matrices."""
    return ref.corpus(500)


@pytest.fixture(scope="session")
def argcsr():
    import paper_1203_5737_b200

    return paper_1203_5737_b200


@pytest.fixture(autouse=True)
def _fresh_options():
    """Tests that flip ARGCSR_* switches (monkeypatch.setenv + reload_options)
    must not leak them: every test starts from the environment as restored by
    the previous test's monkeypatch teardown."""
    try:
        import paper_1203_5737_b200 as m

        m._ext.reload_options()
    except Exception:
        pass
    yield
