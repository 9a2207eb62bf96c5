kernel mm_colmajor {
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let j = tid / N;
  let i = tid % N;
  s = 0;
  for (k = 0; k < N; k++) {
    s += a[i * N + k] * b[k * N + j];
  }
  c[i * N + j] = s;
}
