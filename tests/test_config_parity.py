"""Launch-config reader parity (CPU): veqh_parse_config (the product's
parse_config, include/veq_host.h) against the reference's parse_config
(proj/src/frontend.cpp:1017-1110) run through oracle/_ref/ref_harness, on
valid configs and on every error the reference distinguishes (first failing
line wins, integer overflow vs trailing characters, unknown keys)."""
import ctypes as C
import os
import subprocess
import tempfile

import pytest

from paper_2511_12638_b200 import frontend

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HARNESS = os.path.join(ROOT, "oracle", "_ref", "ref_harness")

CASES = [
    "version = 1\nthreads = 4\ninputs = x\noutputs = y\n",
    "# comment only\n\n  threads=8   # trailing\nwarp_size = 4\nparams.N = -12\nparams.M=+7\n",
    "threads_a = 3\nthreads_b = 5\ninputs = a, b ,c\noutputs=y z\n",
    "params.BIG = 9223372036854775807\nparams.SMALL = -9223372036854775808\n",
    "threads = 1048576\n",
    "threads = 1048577\n",
    "threads = 0\n",
    "threads = 4x\n",
    "threads = -\n",
    "threads = 99999999999999999999\n",
    "version = 2\n",
    "threads\n",
    "threads = \n",
    " = 4\n",
    "params. = 3\n",
    "params.N = 12abc\n",
    "params.N = abc\n",
    "params.N = 99999999999999999999\n",
    "params.N = 99999999999999999999abc\n",
    "params.N = -9223372036854775809\n",
    "colour = blue\n",
    "threads = 4\nparams.N = x\nbogus line\n",
    "threads = 4\nbogus line\nparams.N = x\n",
    "warp_size = 0\n",
    "inputs = x\ninputs = y\nthreads = 2\nthreads = 3\n",
    "threads = 4\r\nparams.K = 2\r\n",
]


def ours(text: str):
    L = frontend._L()
    L.veqh_parse_config.argtypes = [C.c_char_p, C.c_char_p, C.c_size_t]
    L.veqh_parse_config.restype = C.c_int
    buf = C.create_string_buffer(1 << 16)
    st = L.veqh_parse_config(text.encode(), buf, len(buf))
    return st, buf.value.decode()


@pytest.mark.skipif(not os.path.exists(HARNESS), reason="oracle not built")
@pytest.mark.parametrize("i", range(len(CASES)))
def test_parse_config_matches_reference(i):
    text = CASES[i]
    with tempfile.NamedTemporaryFile("w", suffix=".cfg", delete=False) as f:
        f.write(text)
    try:
        r = subprocess.run([HARNESS, "config", f.name], capture_output=True, text=True, timeout=60)
    finally:
        os.unlink(f.name)
    st, out = ours(text)
    assert (st == 0) == (r.returncode == 0), (out, r.stdout)
    assert out == r.stdout


def test_parse_config_error_wording():
    st, out = ours("threads = 4\nparams.N = 1.5\n")
    assert st != 0 and out == "2:1: parameter N must be an integer"
