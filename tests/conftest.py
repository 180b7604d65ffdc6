import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built libhcub_b200.so")
    config.addinivalue_line("markers", "slow: long-running CPU test")


def load_k1(name):
    z = np.load(os.path.join(GOLDEN, f"k1_{name}.npz"))
    out = {k: z[k] for k in z.files}
    out["spec"] = json.loads(str(out["spec"]))
    return out


def load_json(prefix, name):
    with open(os.path.join(GOLDEN, f"{prefix}_{name}.json")) as fh:
        return json.load(fh)


def golden_names(prefix):
    ext = ".npz" if prefix == "k1" else ".json"
    return sorted(f[len(prefix) + 1:-len(ext)] for f in os.listdir(GOLDEN)
                  if f.startswith(prefix + "_") and f.endswith(ext))


def oracle_f(spec):
    from oracle import hcub_oracle as orc
    if spec["f"] == "pp":
        return orc.product_peak(spec["d"], spec.get("center", 0.5), spec.get("sharpness", 50.0))
    return orc.integrand(spec["f"], spec["d"])


def domain_of(spec):
    d = spec["d"]
    if "lo" in spec:
        return np.array(spec["lo"], dtype=float), np.array(spec["hi"], dtype=float)
    return np.zeros(d), np.ones(d)


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN
