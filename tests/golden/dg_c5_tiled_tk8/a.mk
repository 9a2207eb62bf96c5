// C1 reference: one thread per output element, naive k loop.
kernel matmul_rowcol {
  param N;
  in a[N * N];
  in b[N * N];
  out c[N * N];

  let i = tid / N;
  let j = tid % N;
  s = 0;
  for (k = 0; k < N; k++) {
    s += a[i * N + k] * b[k * N + j];
  }
  c[i * N + j] = s;
}
