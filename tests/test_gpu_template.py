"""Device template expansion (veq_load_template + veq_instantiate) against
loading the per-CTA elaborations: identical run results (steps, releases,
faults) and identical canonical nodes in every Out cell, for every CTA of
each grid family, with kernel A's and kernel B's templates merged into one
(program-major expansion: A's instances, then B's)."""
import numpy as np
import pytest

from paper_2511_12638_b200 import frontend, ir, workloads
from paper_2511_12638_b200 import native as N
from paper_2511_12638_b200.engine import Session

pytestmark = pytest.mark.gpu

GRIDS = [
    ("c2", workloads.c2_reduce(n_blocks=6, block=64)),
    ("c3", workloads.c3_conv(2, 3, 8, 12, 4, 4)),
    ("c4", workloads.c4_attention(16, 4, 4, 2, 4)),
    ("c4_tpr1", workloads.c4_attention(12, 2, 2, 1, 4)),
]


def _cells(s, h, batch, nprog):
    out = []
    for p in range(nprog):
        pm = batch.progs[p] if batch is not None else None
        o0 = int(pm["array_off"])
        for k in range(int(pm["n_arrays"])):
            if int(batch.arrays[o0 + k]["role"]) == N.ROLE_OUT:
                out.append(s.fetch_cells(h, p, k, int(batch.arrays[o0 + k]["size"])).tolist())
    return out


@pytest.mark.parametrize("name,w", GRIDS, ids=[g[0] for g in GRIDS])
def test_instantiated_grid_equals_loaded_grid(name, w):
    n = w.n_blocks
    ta, tb, inputs, da, db = frontend.elaborate_template(w.kernel_a, w.kernel_b, w.cfg, w.block_param, n)
    a, b, inp2 = frontend.elaborate_pair(w.kernel_a, w.kernel_b, w.cfg, w.block_param, n)
    assert inputs == inp2
    s = Session(0, max_nodes=1 << 20, max_kid_words=1 << 22, scratch_bytes=256 << 20)
    try:
        s.declare_inputs(inputs)
        merged = ir.concat([a, b])
        h1 = s.load(merged)
        r1 = s.run_raw(h1)
        steps1 = [(r1.progs[p].steps, r1.progs[p].releases, r1.progs[p].n_faults) for p in range(r1.n_progs)]
        c1 = _cells(s, h1, merged, 2 * n)
        t = s.load_template(ir.concat([ta, tb]))
        h2 = s.instantiate(t, np.concatenate([da, db], axis=1))
        r2 = s.run_raw(h2)
        steps2 = [(r2.progs[p].steps, r2.progs[p].releases, r2.progs[p].n_faults) for p in range(r2.n_progs)]
        c2 = _cells(s, h2, merged, 2 * n)  # same per-program array layout
        assert steps1 == steps2
        assert c1 == c2  # same term table: equal canonical forms are equal ids
        s.drop(h1)
        s.drop(h2)
    finally:
        s.close()
