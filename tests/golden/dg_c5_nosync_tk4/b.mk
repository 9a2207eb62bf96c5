kernel mm_nosync {
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
  for (kt = 0; kt < N / TK; kt++) {
    if (tid < N * TK) {
      ta[tid] = a[(tid / TK) * N + kt * TK + tid % TK];
      tb[tid] = b[(kt * TK + tid / N) * N + tid % N];
    }
    
    for (k = 0; k < TK; k++) {
      s += ta[row * TK + k] * tb[k * N + col];
    }
    
  }
  c[row * N + col] = s;
}
