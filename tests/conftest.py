import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built engine")
    config.addinivalue_line("markers", "slow: long-running check")


def load_golden(name):
    with gzip.open(os.path.join(GOLDEN, f"{name}.json.gz"), "rt", encoding="utf-8") as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def golden_pure():
    return load_golden("pure")["data"]


@pytest.fixture(scope="session")
def golden_scenarios():
    return load_golden("scenarios")["data"]


@pytest.fixture(scope="session")
def golden_baseline():
    path = os.path.join(GOLDEN, "baseline.json.gz")
    if not os.path.exists(path):
        pytest.skip("baseline fixture not generated")
    return load_golden("baseline")["data"]


@pytest.fixture(scope="session")
def golden_c5():
    path = os.path.join(GOLDEN, "c5_seed0.json.gz")
    if not os.path.exists(path):
        pytest.skip("c5 fixture not generated")
    return load_golden("c5_seed0")["data"]


@pytest.fixture(scope="session")
def model_dir(tmp_path_factory):
    """The golden model files, uncompressed, as learned-mode configs name them."""
    d = tmp_path_factory.mktemp("models")
    for f in os.listdir(GOLDEN):
        if f.startswith("forest_") and f.endswith(".json.gz") and f != "forest_predictions.json.gz":
            with gzip.open(os.path.join(GOLDEN, f), "rb") as src:
                (d / f[:-3]).write_bytes(src.read())
    return str(d)


@pytest.fixture(scope="session")
def golden_learned():
    return load_golden("learned_scenarios")["data"]


@pytest.fixture(scope="session")
def golden_forest_predictions():
    return load_golden("forest_predictions")["data"]


@pytest.fixture(scope="session")
def engine():
    from paper_2508_03148_b200.engine import Engine
    return Engine(0)
