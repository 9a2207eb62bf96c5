"""Template elaboration (CPU): a grid elaborated ONCE with the block
parameter symbolic, instantiated per CTA by shifting array offsets, must be
byte-identical to elaborating each CTA on its own (veqh_elaborate_grid, the
path pinned against the reference in test_frontend_parity) — for every CTA
of every grid workload family, and grids whose control depends on the block
must be refused (VEQH_E_TEMPLATE) rather than approximated."""
import numpy as np
import pytest

from paper_2511_12638_b200 import frontend, ir, workloads

FIELDS = ("progs", "thread_stmt", "thread_nregs", "stmts", "arrays", "consts", "syncsets", "set_words",
          "thread_reg_off", "locs")


def _same(x, y):
    for f in FIELDS:
        assert np.array_equal(getattr(x, f), getattr(y, f)), f
    assert x.array_names == y.array_names and x.reg_names == y.reg_names and x.prog_names == y.prog_names


GRIDS = [
    ("c2", workloads.c2_reduce(n_blocks=6, block=64)),
    ("c3", workloads.c3_conv(2, 3, 8, 12, 4, 4)),
    ("c3_sq", workloads.c3_conv(3, 2, 8, 8, 2, 2)),
    ("c4", workloads.c4_attention(16, 4, 4, 2, 4)),
    ("c4_tpr1", workloads.c4_attention(12, 2, 2, 1, 4)),
]


@pytest.mark.parametrize("name,w", GRIDS, ids=[g[0] for g in GRIDS])
def test_template_instances_equal_per_cta_elaboration(name, w):
    n = w.n_blocks
    ta, tb, inputs, da, db = frontend.elaborate_template(w.kernel_a, w.kernel_b, w.cfg, w.block_param, n)
    assert da.shape[0] == db.shape[0] == n
    for blk in range(n):
        a, b, inp = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, w.block_param, 1, block_base=blk)
        assert inp == inputs
        _same(ir.instantiate(ta, da[blk]), a)
        _same(ir.instantiate(tb, db[blk]), b)


def test_template_offset_base_and_range():
    w = workloads.c2_reduce(n_blocks=16, block=32)
    ta, tb, inputs, da, db = frontend.elaborate_template(w.kernel_a, w.kernel_b, w.cfg, "B", 5, block_base=9)
    for k in range(5):
        a, b, _ = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, "B", 1, block_base=9 + k)
        _same(ir.instantiate(ta, da[k]), a)
        _same(ir.instantiate(tb, db[k]), b)


BLOCK_CONTROL = """kernel k {
  param B;
  in x[64];
  out y[4];
  if (B < 2) { y[tid] = x[tid]; } else { y[tid] = x[tid] + x[tid + 1]; }
}
"""
BLOCK_CONST = """kernel k {
  param B;
  in x[64];
  out y[4];
  y[tid] = x[tid] * B;
}
"""
NONUNIFORM = """kernel k {
  param B;
  in x[64];
  out y[4];
  y[tid] = x[tid] + x[B * 4 + tid];
}
"""
CFG = "version = 1\nthreads = 4\nparams.B = 0\ninputs = x\noutputs = y\n"


@pytest.mark.parametrize("src", [BLOCK_CONTROL, BLOCK_CONST, NONUNIFORM], ids=["control", "const", "nonuniform"])
def test_block_dependent_grids_are_refused(src):
    with pytest.raises(frontend.TemplateUnsupported):
        frontend.elaborate_template(src, src, CFG, "B", 4)


def test_template_errors_are_the_concrete_errors():
    # B - B is concrete (0) in the template: the division by zero is raised
    # exactly as every CTA's own elaboration raises it
    bad = "kernel k { param B; in x[4]; out y[4]; for (i = 0; i < 3 / (B - B); i++) { } y[tid] = x[tid]; }"
    with pytest.raises(frontend.FrontendError) as e1:
        frontend.elaborate_pair(bad, bad, CFG, "B", 1)
    with pytest.raises(frontend.FrontendError) as e2:
        frontend.elaborate_template(bad, bad, CFG, "B", 2)
    assert "division by zero in static expression" in str(e1.value)
    assert str(e1.value) == str(e2.value) and e1.value.kernel == e2.value.kernel == "a"
