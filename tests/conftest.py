import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden"
FIXTURES = sorted((GOLDEN / "fixtures").iterdir())


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200); runs the sm_100a path")


@pytest.fixture(scope="session")
def port():
    from oracle.bindings import Port
    return Port()


@pytest.fixture(scope="session")
def ref():
    """The reference library compiled from /root/reference sources (oracle/_ref)."""
    from oracle.bindings import REF_SO, RefLib
    if not REF_SO.exists():
        pytest.skip("oracle/_ref/libdemc_ref.so not built (reference sources absent)")
    return RefLib()


@pytest.fixture(scope="session")
def compiler():
    import paper_2604_16613_b200 as gp
    return gp.Compiler(0)


def fixture_case(path: Path):
    import paper_2604_16613_b200 as gp
    from oracle.bindings import parse_dem_text
    circuit = gp.parse_circuit((path / "circuit.txt").read_text())
    level = int((path / "level").read_text())
    text = (path / "expected.dem").read_text()
    return circuit, level, text, parse_dem_text(text)
