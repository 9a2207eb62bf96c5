"""Frontend parity (CPU): the product frontend (libveq_host.so) must produce
byte-identical packed IR to the reference frontend's elaboration, as dumped
by the oracle (tests/golden/*/{a,b}.veqir): same statements, registers,
constant and sync-set pools, array table, register names and source
locations. Kernel sources are read from the reference corpus when it is
mounted (build container); the test is skipped elsewhere."""
import json
import os

import numpy as np
import pytest

from conftest import golden_dirs
from paper_2511_12638_b200 import frontend, ir

KDIR = "/root/reference/proj/kernels"


def _manifest_rows():
    path = os.path.join(KDIR, "manifest.txt")
    if not os.path.exists(path):
        return []
    rows = []
    for line in open(path):
        line = line.strip()
        if line and not line.startswith("#"):
            rows.append(line.split()[:3])
    return rows


def _same(x: ir.Batch, y: ir.Batch):
    for f in ("progs", "thread_stmt", "thread_nregs", "stmts", "arrays", "consts", "syncsets", "set_words",
              "thread_reg_off", "locs"):
        assert np.array_equal(getattr(x, f), getattr(y, f)), f
    assert x.array_names == y.array_names
    assert x.reg_names == y.reg_names
    assert x.prog_names == y.prog_names


@pytest.mark.skipif(not os.path.isdir(KDIR), reason="reference corpus not mounted")
@pytest.mark.parametrize("i", range(15))
def test_corpus_elaboration_identical(i):
    rows = _manifest_rows()
    ka, kb, cfg = rows[i]
    d = golden_dirs(f"corpus_{i:02d}_")[0]
    g = json.load(open(os.path.join(d, "golden.json")))
    src = lambda f: open(os.path.join(KDIR, f)).read()
    if "elab_error" in g:
        with pytest.raises(frontend.FrontendError):
            frontend.elaborate_pair(src(ka), src(kb), src(cfg))
        return
    a, b, inputs = frontend.elaborate_pair(src(ka), src(kb), src(cfg))
    assert inputs == [(x["name"], x["size"]) for x in g["inputs"]]
    _same(a, ir.load(os.path.join(d, "a.veqir")))
    _same(b, ir.load(os.path.join(d, "b.veqir")))


def test_frontend_errors_match_reference_wording():
    bad = "kernel k { in x[4]; out y[4]; y[tid] = x[tid] $ 1; }"
    with pytest.raises(frontend.FrontendError) as e:
        frontend.elaborate_pair(bad, bad, "version = 1\nthreads = 4\ninputs = x\noutputs = y\n")
    assert e.value.kernel == "a"
    assert "unexpected character '$'" in str(e.value)
    dd = "kernel k { in x[4]; out y[4]; y[x[0]] = 1; }"
    with pytest.raises(frontend.FrontendError) as e:
        frontend.elaborate_pair(dd, dd, "version = 1\nthreads = 4\ninputs = x\noutputs = y\n")
    assert "data-dependent address: array element x[...] is a runtime value" in str(e.value)


@pytest.mark.parametrize("d", golden_dirs("wl_"), ids=os.path.basename)
def test_workload_elaboration_identical(d):
    """Our benchmark kernels (fixture dirs hold the sources) elaborate exactly
    as the reference elaborated them."""
    src = lambda f: open(os.path.join(d, f)).read()
    a, b, inputs = frontend.elaborate_pair(src("a.mk"), src("b.mk"), src("cfg.cfg"))
    g = json.load(open(os.path.join(d, "golden.json")))
    assert inputs == [(x["name"], x["size"]) for x in g["inputs"]]
    _same(a, ir.load(os.path.join(d, "a.veqir")))
    _same(b, ir.load(os.path.join(d, "b.veqir")))
