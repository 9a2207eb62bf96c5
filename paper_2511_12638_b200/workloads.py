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
  C3 conv 3x3: direct vs im2col-tiled, a grid of pixel tiles
  C4 attention: naive softmax(QK^T)V with row-max subtraction vs blocked
     online softmax (FlashAttention-style rescaling), a grid of query blocks
  C5 matmul variants vs one reference: a seeded mutation generator; each
     variant is its own CTA pair, and a batch holds many variants
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Tuple


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


# ---------------------------------------------------------------- C3 -------
def c3_conv(cin: int = 64, cout: int = 64, h: int = 256, w: int = 256, th: int = 16, tw: int = 16) -> Workload:
    """3x3 convolution, stride 1, on a pre-padded input x[cin][h+2][w+2];
    one CTA per th x tw output tile (block index B, row-major over tiles),
    one thread per output pixel computing every output channel. Each CTA's
    Out array is its own tile y[co][pixel] (the reference checks one CTA and
    requires every Out cell written, pipeline.cpp:73-87)."""
    tiles_w = w // tw
    hp, wp = h + 2, w + 2
    direct = f"""// C3 reference: direct 3x3 convolution, one thread per output pixel.
kernel conv_direct {{
  param B;
  param CI;
  param CO;
  param H;
  param W;
  param TH;
  param TW;
  param TWS;
  in x[CI * (H + 2) * (W + 2)];
  in wt[CO * CI * 9];
  out y[CO * TH * TW];

  let oh = (B / TWS) * TH + tid / TW;
  let ow = (B % TWS) * TW + tid % TW;
  for (co = 0; co < CO; co++) {{
    s = 0;
    for (ci = 0; ci < CI; ci++) {{
      for (kh = 0; kh < 3; kh++) {{
        for (kw = 0; kw < 3; kw++) {{
          s += x[(ci * (H + 2) + oh + kh) * (W + 2) + ow + kw] * wt[(co * CI + ci) * 9 + kh * 3 + kw];
        }}
      }}
    }}
    y[co * TH * TW + tid] = s;
  }}
}}
"""
    im2col = f"""// C3 candidate: im2col. Each thread stages its pixel's 3x3xCI patch as a
// column of the shared patch matrix, a barrier, then a K = 9*CI GEMM
// against the filter rows.
kernel conv_im2col {{
  param B;
  param CI;
  param CO;
  param H;
  param W;
  param TH;
  param TW;
  param TWS;
  in x[CI * (H + 2) * (W + 2)];
  in wt[CO * CI * 9];
  out y[CO * TH * TW];
  scratch col[CI * 9 * TH * TW];

  let oh = (B / TWS) * TH + tid / TW;
  let ow = (B % TWS) * TW + tid % TW;
  for (k = 0; k < CI * 9; k++) {{
    col[k * TH * TW + tid] = x[((k / 9) * (H + 2) + oh + (k % 9) / 3) * (W + 2) + ow + k % 3];
  }}
  sync;
  for (co = 0; co < CO; co++) {{
    acc = 0;
    for (k = 0; k < CI * 9; k++) {{
      acc += wt[co * CI * 9 + k] * col[k * TH * TW + tid];
    }}
    y[co * TH * TW + tid] = acc;
  }}
}}
"""
    cfg = f"""version = 1
threads = {th * tw}
params.B = 0
params.CI = {cin}
params.CO = {cout}
params.H = {h}
params.W = {w}
params.TH = {th}
params.TW = {tw}
params.TWS = {tiles_w}
inputs = x, wt
outputs = y
"""
    n_tiles = (h // th) * tiles_w
    return Workload("c3_conv", direct, im2col, cfg, n_tiles, "B", cout * th * tw)


# ---------------------------------------------------------------- C4 -------
def c4_attention(seq: int = 4096, d: int = 128, rows: int = 16, tpr: int = 16, bc: int = 64) -> Workload:
    """One head, Q/K/V [seq][d]. One CTA per block of `rows` query rows
    (block index B), `tpr` threads per row. A: scores of the whole row in
    scratch, row max, p = exp(s - m), denominator, o = (sum p v) / den.
    B: online softmax over key blocks of `bc` rows — per block the running
    max m, rescale c = exp(m - m'), running denominator and accumulators
    (FlashAttention-style); block 0 seeds the state. Both subtract the row
    max, so their canonical forms coincide. Each CTA's
    Out array is its own rows o[r][e]."""
    naive = f"""// C4 reference: naive attention, row max subtracted before exp.
kernel attn_naive {{
  param B;
  param L;
  param D;
  param R;
  param TPR;
  in q[L * D];
  in kmat[L * D];
  in vmat[L * D];
  out o[R * D];
  scratch sc[R * L];
  scratch mx[R];
  scratch den[R];

  let r = tid / TPR;
  let j = tid % TPR;
  let qr = B * R + r;
  for (l = j; l < L; l += TPR) {{
    acc = 0;
    for (e = 0; e < D; e++) {{
      acc += q[qr * D + e] * kmat[l * D + e];
    }}
    sc[r * L + l] = acc;
  }}
  sync;
  if (j == 0) {{
    m = NEG_INF;
    for (l = 0; l < L; l++) {{
      m = max(m, sc[r * L + l]);
    }}
    mx[r] = m;
  }}
  sync;
  for (l = j; l < L; l += TPR) {{
    sc[r * L + l] = exp(sc[r * L + l] - mx[r]);
  }}
  sync;
  if (j == 0) {{
    dn = 0;
    for (l = 0; l < L; l++) {{
      dn += sc[r * L + l];
    }}
    den[r] = dn;
  }}
  sync;
  for (e = j; e < D; e += TPR) {{
    acc = 0;
    for (l = 0; l < L; l++) {{
      acc += sc[r * L + l] * vmat[l * D + e];
    }}
    o[r * D + e] = acc / den[r];
  }}
}}
"""
    online = f"""// C4 candidate: online softmax over key blocks of BC rows.
kernel attn_online {{
  param B;
  param L;
  param D;
  param R;
  param TPR;
  param BC;
  in q[L * D];
  in kmat[L * D];
  in vmat[L * D];
  out o[R * D];
  scratch sb[R * BC];
  scratch ms[R];
  scratch cs[R];
  scratch ds[R];
  scratch oa[R * D];

  let r = tid / TPR;
  let j = tid % TPR;
  let qr = B * R + r;
  for (kb = 0; kb < L / BC; kb++) {{
    for (l = j; l < BC; l += TPR) {{
      acc = 0;
      for (e = 0; e < D; e++) {{
        acc += q[qr * D + e] * kmat[(kb * BC + l) * D + e];
      }}
      sb[r * BC + l] = acc;
    }}
    sync;
    if (j == 0) {{
      if (kb == 0) {{
        m = NEG_INF;
      }} else {{
        m = ms[r];
      }}
      mn = m;
      for (l = 0; l < BC; l++) {{
        mn = max(mn, sb[r * BC + l]);
      }}
      if (kb == 0) {{
        dn = 0;
      }} else {{
        c = exp(m - mn);
        cs[r] = c;
        dn = ds[r] * c;
      }}
      for (l = 0; l < BC; l++) {{
        pl = exp(sb[r * BC + l] - mn);
        sb[r * BC + l] = pl;
        dn += pl;
      }}
      ms[r] = mn;
      ds[r] = dn;
    }}
    sync;
    for (e = j; e < D; e += TPR) {{
      if (kb == 0) {{
        acc = 0;
      }} else {{
        acc = oa[r * D + e] * cs[r];
      }}
      for (l = 0; l < BC; l++) {{
        acc += sb[r * BC + l] * vmat[(kb * BC + l) * D + e];
      }}
      oa[r * D + e] = acc;
    }}
    sync;
  }}
  for (e = j; e < D; e += TPR) {{
    o[r * D + e] = oa[r * D + e] / ds[r];
  }}
}}
"""
    cfg = f"""version = 1
threads = {rows * tpr}
params.B = 0
params.L = {seq}
params.D = {d}
params.R = {rows}
params.TPR = {tpr}
params.BC = {bc}
inputs = q, kmat, vmat
outputs = o
"""
    return Workload("c4_attention", naive, online, cfg, seq // rows, "B", rows * d)


# ---------------------------------------------------------------- C5 -------
C5_SEED = 20261017
C5_KINDS = ("tiled", "colmajor", "reverse_k", "unroll2", "nosync", "index_bug", "wrong_guard", "oob")


def _c5_variant(kind: str, n: int, tk: int) -> str:
    """One mutated matmul kernel (n x n x n, one thread per output)."""
    idx = "(k + 1) % N" if kind == "index_bug" else "k"
    lo = "1" if kind == "wrong_guard" else "0"
    if kind in ("tiled", "nosync"):
        sync = "" if kind == "nosync" else "sync;"
        return f"""kernel mm_{kind} {{
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
    {sync}
    for (k = 0; k < TK; k++) {{
      s += ta[row * TK + k] * tb[k * N + col];
    }}
    {sync}
  }}
  c[row * N + col] = s;
}}
"""
    if kind == "colmajor":
        ij = "let j = tid / N;\n  let i = tid % N;"
    else:
        ij = "let i = tid / N;\n  let j = tid % N;"
    if kind == "reverse_k":
        loop = "for (kk = 0; kk < N; kk++) {\n    s += a[i * N + N - 1 - kk] * b[(N - 1 - kk) * N + j];\n  }"
    elif kind == "unroll2":
        loop = ("for (k = 0; k < N; k += 2) {\n    s += a[i * N + k] * b[k * N + j];\n"
                "    s += a[i * N + k + 1] * b[(k + 1) * N + j];\n  }")
    elif kind == "oob":
        loop = "for (k = 0; k < N; k++) {\n    s += a[i * N + k + 1] * b[k * N + j];\n  }"
    else:
        loop = f"for (k = {lo}; k < N; k++) {{\n    s += a[i * N + k] * b[{idx} * N + j];\n  }}"
    return f"""kernel mm_{kind} {{
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  {ij}
  s = 0;
  {loop}
  c[i * N + j] = s;
}}
"""


def c5_variants(n_variants: int = 1000, n: int = 32, seed: int = C5_SEED) -> List[Tuple[str, str, str]]:
    """(kind, kernel source, cfg) per variant, from a seeded generator:
    ~70% semantics-preserving (tiling with TK in {1,2,4,8,16,32} clipped to
    N, column-major thread mapping, reversed k, unroll by 2), 10% dropped
    barrier (race), 10% index bug (not equivalent), 5% wrong loop guard,
    5% out-of-bounds read. The reference kernel is
    c1_matmul's per-thread naive form at the same N."""
    import random
    rng = random.Random(seed)
    out = []
    tks = [t for t in (1, 2, 4, 8, 16, 32) if t <= n and n % t == 0]
    for _ in range(n_variants):
        u = rng.random()
        if u < 0.70:
            kind = rng.choice(["tiled", "colmajor", "reverse_k", "unroll2"])
        elif u < 0.80:
            kind = "nosync"
        elif u < 0.90:
            kind = "index_bug"
        elif u < 0.95:
            kind = "wrong_guard"
        else:
            kind = "oob"
        tk = rng.choice(tks)
        cfg = f"""version = 1
threads = {n * n}
params.N = {n}
params.TK = {tk}
inputs = a, b
outputs = c
"""
        out.append((kind, _c5_variant(kind, n, tk), cfg))
    return out


def c5_reference(n: int = 32) -> str:
    return c1_matmul(n).kernel_a


WORKLOADS = {"c1_matmul": c1_matmul, "c2_reduce": c2_reduce, "c3_conv": c3_conv, "c4_attention": c4_attention}
