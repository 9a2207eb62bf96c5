import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_dirs(prefix=""):
    out = []
    for d in sorted(os.listdir(GOLDEN)):
        p = os.path.join(GOLDEN, d)
        if os.path.isdir(p) and d.startswith(prefix) and (
                os.path.exists(os.path.join(p, "golden.json")) or os.path.exists(os.path.join(p, "golden.json.gz"))):
            out.append(p)
    return out


def load_golden(d):
    """A fixture's golden.json (or its gzipped form, golden.json.gz)."""
    p = os.path.join(d, "golden.json")
    if os.path.exists(p):
        return json.load(open(p))
    with gzip.open(p + ".gz", "rt") as f:
        return json.load(f)


def gen_dirs():
    g = os.path.join(GOLDEN, "gen")
    return sorted(os.path.join(g, d) for d in os.listdir(g)) if os.path.isdir(g) else []


@pytest.fixture(scope="session")
def session():
    from paper_2511_12638_b200.engine import Session
    s = Session(0, max_nodes=1 << 20, max_kid_words=1 << 22, scratch_bytes=256 << 20, keep_regs=True)
    yield s
    s.close()
