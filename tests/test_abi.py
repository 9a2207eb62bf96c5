"""C-ABI boundary (CPU): both libraries load and export every function their
headers declare (include/veq.h, include/veq_host.h), the Python mirror
binds them all, and — with no GPU — the product path fails loudly
(VEQ_E_NO_DEVICE) instead of falling back to a CPU implementation."""
import ctypes
import os
import re

import pytest

from paper_2511_12638_b200 import frontend, native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?[a-z_0-9]+\s*\**\s*(veqh?_[a-z_0-9]+)\s*\(", src, flags=re.M)))


def test_veq_h_exports():
    names = _declared("veq.h")
    assert "veq_run" in names and "veq_compare" in names and len(names) >= 14
    lib = ctypes.CDLL(native.LIB_PATH)
    for n in names:
        assert hasattr(lib, n), n
    assert set(names) <= set(native.EXPORTED), set(names) - set(native.EXPORTED)


def test_veq_host_h_exports():
    names = _declared("veq_host.h")
    assert {"veqh_elaborate_grid", "veqh_free", "veqh_parse_config"} <= set(names)
    lib = ctypes.CDLL(frontend.HOST_LIB)
    for n in names:
        assert hasattr(lib, n), n


def test_strerror_table():
    L = native.lib()
    assert L.veq_strerror(0).decode() == "ok"
    assert "capacity" in L.veq_strerror(1).decode()
    assert L.veq_strerror(8).decode() == "no CUDA device"


@pytest.mark.skipif(__import__("torch").cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_device_fails_loudly():
    from paper_2511_12638_b200.engine import Session
    with pytest.raises(native.VeqError) as e:
        Session(0)
    assert e.value.status == 8
