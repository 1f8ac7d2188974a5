import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if REPO not in sys.path:
    sys.path.insert(0, REPO)

GOLDEN_DIR = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA engine)")
    config.addinivalue_line("markers", "slow: long-running (full-size configs)")


class Golden:
    """Reference outputs recorded by tests/golden/make_golden.py from the unmodified oocdet."""

    def __init__(self):
        with open(os.path.join(GOLDEN_DIR, "manifest.json")) as f:
            self.manifest = json.load(f)
        self.arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
        self.cases = self.manifest["cases"]
        self.tables = self.manifest["tables"]

    def input(self, name):
        key = f"{name}__input"
        if key in self.arrays:
            return self.arrays[key]
        from paper_2503_04424_b200 import gen

        regen = {
            "C1": lambda: gen.spd_wishart(4096, 4096, seed=0, shift=1e-3),
            "rbf512": lambda: gen.rbf(512, seed=41),
            "ntk384": lambda: gen.ntk_like(384, 768, 0.75, seed=42),
        }
        return regen[name]()

    def run(self, name, key):
        meta = self.cases[name]["runs"][key]
        out = dict(meta)
        for field in ("prefix", "perm", "signs"):
            k = f"{name}__{key}__{field}"
            if k in self.arrays:
                out[field] = self.arrays[k]
        return out


@pytest.fixture(scope="session")
def golden():
    return Golden()


def rel_err(x, ref):
    x = np.asarray(x, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    return float(np.max(np.abs(x - ref) / np.maximum(1.0, np.abs(ref)))) if len(ref) else 0.0
