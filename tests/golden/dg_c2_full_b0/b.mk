// C2 candidate: warp-shuffle tree reduction of a CTA's slice. Each
// __shfl_down is modelled as a store to scratch, a warp barrier, a load of
// the partner lane and a second warp barrier; warp leaders publish partials
// behind a block barrier and warp 0 reduces them.
kernel reduce_shfl {
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
  sh[tid] = v;
  syncwarp(w);
  if (lane < 16) { v = v + sh[tid + 16]; }
  syncwarp(w);
  sh[tid] = v;
  syncwarp(w);
  if (lane < 24) { v = v + sh[tid + 8]; }
  syncwarp(w);
  sh[tid] = v;
  syncwarp(w);
  if (lane < 28) { v = v + sh[tid + 4]; }
  syncwarp(w);
  sh[tid] = v;
  syncwarp(w);
  if (lane < 30) { v = v + sh[tid + 2]; }
  syncwarp(w);
  sh[tid] = v;
  syncwarp(w);
  if (lane < 31) { v = v + sh[tid + 1]; }
  syncwarp(w);
  if (lane == 0) {
    part[w] = v;
  }
  sync;
  if (w == 0) {
    if (lane < BS / 32) {
      v = part[lane];
    } else {
      v = 0;
    }
    sh[tid] = v;
    syncwarp(w);
    if (lane < 16) { v = v + sh[tid + 16]; }
    syncwarp(w);
    sh[tid] = v;
    syncwarp(w);
    if (lane < 24) { v = v + sh[tid + 8]; }
    syncwarp(w);
    sh[tid] = v;
    syncwarp(w);
    if (lane < 28) { v = v + sh[tid + 4]; }
    syncwarp(w);
    sh[tid] = v;
    syncwarp(w);
    if (lane < 30) { v = v + sh[tid + 2]; }
    syncwarp(w);
    sh[tid] = v;
    syncwarp(w);
    if (lane < 31) { v = v + sh[tid + 1]; }
    syncwarp(w);
    if (tid == 0) {
      y[0] = v;
    }
  }
}
