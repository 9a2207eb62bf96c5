"""Error paths of the C-ABI: capacity, exact-range and
envelope errors are status codes, never silent truncation or rounding.

- VEQ_E_BUDGET: the term table's capacity is exhausted (the reference's
  BudgetError maps here, CLI exit 4, proj/tools/main.cpp:419-422);
- VEQ_E_RATIONAL_OVERFLOW: a coefficient leaves the exact int64 range (the
  reference's GMP rationals are unbounded; here the run fails loudly);
- VEQ_E_SCRATCH: a per-node canonicalisation scratch request exceeds the
  pool;
- VEQ_E_UNSUPPORTED: input names whose "<name>_" prefixes interleave in byte
  order (one is a proper prefix of the other) are rejected at declaration.
After each error the context stays usable: clearing the term table and
running a small pair again gives the reference's result."""
import pytest

from paper_2511_12638_b200 import frontend
from paper_2511_12638_b200 import native as N
from paper_2511_12638_b200.engine import Session

pytestmark = pytest.mark.gpu

SUM = """kernel sum_{n} {{
  in x[{n}];
  out y[1];
  s = 0;
  for (i = 0; i < {n}; i++) {{
    s += x[i] * x[{n} - 1 - i];
  }}
  y[0] = s;
}}
"""

BIG = """kernel big {
  in x[4];
  out y[4];
  t = x[tid] * 4000000000;
  t = t * 4000000000;
  t = t * 4000000000;
  y[tid] = t;
}
"""

IDENT = """kernel ident {
  in x[4];
  out y[4];
  y[tid] = x[tid];
}
"""


def _cfg(threads, inputs="x", outputs="y"):
    return f"version = 1\nthreads = {threads}\ninputs = {inputs}\noutputs = {outputs}\n"


def _run(s, src_a, src_b, cfg):
    a, b, inputs = frontend.elaborate_pair(src_a, src_b, cfg)
    s.declare_inputs(inputs)
    return s.run_pair_raw(s.load(a), s.load(b))


def _still_usable(s):
    assert N.lib().veq_clear_terms(s.ctx) == 0
    oa, ob = _run(s, IDENT, IDENT, _cfg(4))
    assert oa.n_faults == 0 and ob.n_faults == 0


def test_budget_is_a_status():
    s = Session(0, max_nodes=1 << 10, max_kid_words=1 << 16, scratch_bytes=64 << 20)
    try:
        src = SUM.format(n=2048)
        with pytest.raises(N.VeqError) as e:
            _run(s, src, src, _cfg(1))
        assert e.value.status == N.E_BUDGET
    finally:
        s.close()


def test_rational_overflow_is_a_status():
    s = Session(0, max_nodes=1 << 16, max_kid_words=1 << 18, scratch_bytes=64 << 20)
    try:
        with pytest.raises(N.VeqError) as e:
            _run(s, BIG, BIG, _cfg(4))
        assert e.value.status == N.E_RATIONAL_OVERFLOW
        _still_usable(s)
    finally:
        s.close()


def test_scratch_is_a_status():
    # a 40,000-term sum canonicalised with a 256 KiB scratch pool
    s = Session(0, max_nodes=1 << 20, max_kid_words=1 << 22, scratch_bytes=256 << 10)
    try:
        src = SUM.format(n=40000)
        with pytest.raises(N.VeqError) as e:
            _run(s, src, src, _cfg(1))
        assert e.value.status == N.E_SCRATCH
        _still_usable(s)
    finally:
        s.close()


def test_interleaved_input_names_rejected():
    s = Session(0, max_nodes=1 << 16, max_kid_words=1 << 18, scratch_bytes=64 << 20)
    try:
        with pytest.raises(N.VeqError) as e:
            s.declare_inputs([("x", 4), ("x_1", 4)])
        assert e.value.status == N.E_UNSUPPORTED
        s.declare_inputs([("x", 4)])
        oa, ob = s.run_pair_raw(*[s.load(b) for b in frontend.elaborate_pair(IDENT, IDENT, _cfg(4))[:2]])
        assert oa.n_faults == 0
    finally:
        s.close()
