"""Synthetic kernel pairs of BASELINE.json's five configurations.

Each workload is a pair of kernels in the reference's kernel language plus a
launch configuration. Multi-CTA configurations are grids: one CTA program per
block, the block index bound to `params.B`, every CTA reading the global
input arrays (so input symbols differ between CTAs) and writing its own
outputs. Shapes follow SURVEY.md §8(d); `scale` shrinks them for parity tests
that the CPU reference must finish in seconds.

  C1 matmul 64x64x64: per-thread naive (4096 thr) vs shared-memory tiled
  C2 reduction 2^20 = 1024 CTAs x 1024: sequential sum (1 thr) vs warp-shuffle
     tree (1024 thr, warp 32; shuffles modelled as store + syncwarp + load)
  C3 conv 3x3: direct vs im2col-tiled (reduced shapes at scale < 1)
  C5 1000 matmul variants vs one reference (variant = its own pair)
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional


@dataclass
class Workload:
    name: str
    kernel_a: str
    kernel_b: str
    cfg: str
    n_blocks: int = 1
    block_param: Optional[str] = None
    elements_per_block: int = 1   # output elements (VCs) per CTA pair

    @property
    def elements(self) -> int:
        return self.n_blocks * self.elements_per_block


# ---------------------------------------------------------------- C2 -------
def _shfl_levels(indent: str, reg: str) -> str:
    """Five warp-shuffle-down levels on scratch `sh`, one syncwarp pair each."""
    out = []
    for off in (16, 8, 4, 2, 1):
        out.append(f"{indent}sh[tid] = {reg};")
        out.append(f"{indent}syncwarp(w);")
        out.append(f"{indent}if (lane < {32 - off}) {{ {reg} = {reg} + sh[tid + {off}]; }}")
        out.append(f"{indent}syncwarp(w);")
    return "\n".join(out)


def c2_reduce(n_blocks: int = 1024, block: int = 1024) -> Workload:
    n = n_blocks * block
    seq = f"""// C2 reference: one thread folds its CTA's slice left to right.
kernel reduce_seq {{
  param B;
  param BS;
  param N;
  in x[N];
  out y[1];

  s = 0;
  for (i = 0; i < BS; i++) {{
    s += x[B * BS + i];
  }}
  y[0] = s;
}}
"""
    tree = f"""// C2 candidate: warp-shuffle tree reduction of a CTA's slice. Each
// __shfl_down is modelled as a store to scratch, a warp barrier, a load of
// the partner lane and a second warp barrier; warp leaders publish partials
// behind a block barrier and warp 0 reduces them.
kernel reduce_shfl {{
  param B;
  param BS;
  param N;
  in x[N];
  out y[1];
  scratch sh[BS];
  scratch part[BS / 32];

  let lane = tid % 32;
  let w = tid / 32;
  v = x[B * BS + tid];
{_shfl_levels("  ", "v")}
  if (lane == 0) {{
    part[w] = v;
  }}
  sync;
  if (w == 0) {{
    if (lane < BS / 32) {{
      v = part[lane];
    }} else {{
      v = 0;
    }}
{_shfl_levels("    ", "v")}
    if (tid == 0) {{
      y[0] = v;
    }}
  }}
}}
"""
    cfg = f"""version = 1
threads_a = 1
threads_b = {block}
warp_size = 32
params.B = 0
params.BS = {block}
params.N = {n}
inputs = x
outputs = y
"""
    return Workload("c2_reduce", seq, tree, cfg, n_blocks, "B", 1)


# ---------------------------------------------------------------- C1 -------
def c1_matmul(n: int = 64, tk: int = 8) -> Workload:
    naive = f"""// C1 reference: one thread per output element, naive k loop.
kernel matmul_rowcol {{
  param N;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let i = tid / N;
  let j = tid % N;
  s = 0;
  for (k = 0; k < N; k++) {{
    s += a[i * N + k] * b[k * N + j];
  }}
  c[i * N + j] = s;
}}
"""
    tiled = f"""// C1 candidate: shared-memory tiled matmul, N*TK slabs of a and b per pass.
kernel matmul_smem {{
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];
  scratch ta[N * TK];
  scratch tb[TK * N];

  let row = tid / N;
  let col = tid % N;
  s = 0;
  for (kt = 0; kt < N / TK; kt++) {{
    if (tid < N * TK) {{
      ta[tid] = a[(tid / TK) * N + kt * TK + tid % TK];
      tb[tid] = b[(kt * TK + tid / N) * N + tid % N];
    }}
    sync;
    for (k = 0; k < TK; k++) {{
      s += ta[row * TK + k] * tb[k * N + col];
    }}
    sync;
  }}
  c[row * N + col] = s;
}}
"""
    cfg = f"""version = 1
threads = {n * n}
params.N = {n}
params.TK = {tk}
inputs = a, b
outputs = c
"""
    return Workload("c1_matmul", naive, tiled, cfg, 1, None, n * n)


WORKLOADS = {"c1_matmul": c1_matmul, "c2_reduce": c2_reduce}
