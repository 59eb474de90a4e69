import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running (skipped unless -m slow)")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name))


def golden_json(name):
    with open(os.path.join(GOLDEN, name)) as fh:
        return json.load(fh)


def model_golden(name):
    """Unpack tests/golden/model_<name>.npz into (cfg, state, dict-of-arrays)."""
    from paper_2604_07239_b200.config import ModelConfig
    from oracle.model import PARAM_ORDER
    z = load_golden(f"model_{name}.npz")
    cfgd = json.loads(bytes(z["cfg_json"]).decode())
    cfg = ModelConfig(**cfgd)
    state = {
        "params": {k: z["p_" + k] for k in PARAM_ORDER},
        "cache": z["cache"],
        "m": [z["m_" + k] for k in PARAM_ORDER],
        "v": [z["v_" + k] for k in PARAM_ORDER],
        "t": int(z["t"]),
        "step_count": int(z["step_count"]),
    }
    return cfg, state, z


@pytest.fixture(scope="session")
def golden():
    return load_golden
