import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line(
        "markers", "gpu: needs a B200 (runs the CUDA decode path)")


@pytest.fixture(scope="session")
def golden_dir():
    return GOLDEN


@pytest.fixture(scope="session")
def manifest():
    import json
    with open(os.path.join(GOLDEN, "manifest.json")) as fh:
        return json.load(fh)


@pytest.fixture(scope="session")
def decode_cases():
    return dict(np.load(os.path.join(GOLDEN, "decode_cases.npz")))


@pytest.fixture(scope="session")
def rng():
    return np.random.default_rng(1234)


def case_calls(cases: dict, name: str):
    """Decode calls recorded for one golden file, in recorded order."""
    idx = sorted({int(k.split("|")[1]) for k in cases if k.startswith(name + "|")})
    out = []
    for i in idx:
        key = f"{name}|{i}"
        c = {"kind": str(cases[key + "|kind"]), "frame": int(cases[key + "|frame"]),
             "pixels": cases[key + "|pixels"],
             "footprint": cases[key + "|footprint"],
             "stats": tuple(int(v) for v in cases[key + "|stats"])}
        c["mask_packed"] = cases.get(key + "|mask")
        if key + "|fractions" in cases:
            c["fractions"] = tuple(float(v) for v in cases[key + "|fractions"])
            c["gaze"] = tuple(float(v) for v in cases[key + "|gaze"])
        out.append(c)
    return out


def unpack_mask(packed, shape):
    n = shape[0] * shape[1]
    return np.unpackbits(packed)[:n].reshape(shape).astype(bool)
