"""The C++ binding of INTEGRATION.md, compiled and run (GPU): the reference
checker's own objects linked with libveq.so (oracle/integration_check.cpp).
check_equivalence is re-stated with run() replaced by the C-ABI (veq_run +
veq_run_report + DAG import into reference Expr objects) and eq()'s fast
path replaced by veq_compare (the reference's slow path decides canonically
different VCs on the imported forms). Its report_to_json must equal the
reference's own report, byte for byte minus timings, on every corpus pair
(the 15 manifest verdicts), every extra pair and every workload fixture."""
import os
import subprocess

import pytest

from conftest import golden_dirs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "oracle", "_ref", "integration_check")


@pytest.mark.gpu
def test_cxx_binding_reproduces_reference_reports():
    if not os.path.exists(EXE):
        pytest.fail("oracle/_ref/integration_check not built (make -C oracle integration)")
    dirs = golden_dirs("corpus_") + golden_dirs("extra_") + golden_dirs("wl_")
    r = subprocess.run([EXE, "--golden"] + dirs, capture_output=True, text=True, timeout=1800)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert r.stdout.strip().splitlines()[-1].startswith("OK")
    n_match = sum(1 for line in r.stdout.splitlines() if line.startswith("MATCH") and "/corpus_" in line)
    assert n_match >= 12  # corpus pairs that reach the hot path (the rest fail in the frontend)
