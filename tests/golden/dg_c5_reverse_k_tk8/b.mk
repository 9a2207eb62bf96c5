kernel mm_reverse_k {
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let i = tid / N;
  let j = tid % N;
  s = 0;
  for (kk = 0; kk < N; kk++) {
    s += a[i * N + N - 1 - kk] * b[(N - 1 - kk) * N + j];
  }
  c[i * N + j] = s;
}
