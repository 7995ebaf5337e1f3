import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parents[1]
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))
GOLD = ROOT / "tests" / "golden"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs under gpurun / the round-end GPU tier)")


@pytest.fixture(scope="session")
def cfg():
    from paper_2211_13939_b200.domain import PipelineConfig
    return PipelineConfig()


@pytest.fixture(scope="session")
def lexicon():
    from paper_2211_13939_b200.frontend import default_lexicon
    return default_lexicon()


@pytest.fixture(scope="session")
def texts():
    from paper_2211_13939_b200.frontend import default_texts
    return default_texts()


@pytest.fixture(scope="session")
def golden_units():
    return dict(np.load(GOLD / "tier_s_units.npz"))


@pytest.fixture(scope="session")
def golden_synth():
    return dict(np.load(GOLD / "tier_s_synth.npz"))


@pytest.fixture(scope="session")
def golden_frontend():
    return json.loads((GOLD / "frontend.json").read_text("utf-8"))


@pytest.fixture(scope="session")
def golden_schedules():
    return json.loads((GOLD / "schedules.json").read_text("utf-8"))
