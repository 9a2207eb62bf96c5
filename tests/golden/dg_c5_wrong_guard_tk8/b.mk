kernel mm_wrong_guard {
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let i = tid / N;
  let j = tid % N;
  s = 0;
  for (k = 1; k < N; k++) {
    s += a[i * N + k] * b[k * N + j];
  }
  c[i * N + j] = s;
}
