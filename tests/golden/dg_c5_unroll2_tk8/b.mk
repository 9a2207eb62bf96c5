kernel mm_unroll2 {
  param N;
  param TK;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let i = tid / N;
  let j = tid % N;
  s = 0;
  for (k = 0; k < N; k += 2) {
    s += a[i * N + k] * b[k * N + j];
    s += a[i * N + k + 1] * b[(k + 1) * N + j];
  }
  c[i * N + j] = s;
}
