// C4 reference: naive attention, row max subtracted before exp.
kernel attn_naive {
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
  for (l = j; l < L; l += TPR) {
    acc = 0;
    for (e = 0; e < D; e++) {
      acc += q[qr * D + e] * kmat[l * D + e];
    }
    sc[r * L + l] = acc;
  }
  sync;
  if (j == 0) {
    m = NEG_INF;
    for (l = 0; l < L; l++) {
      m = max(m, sc[r * L + l]);
    }
    mx[r] = m;
  }
  sync;
  for (l = j; l < L; l += TPR) {
    sc[r * L + l] = exp(sc[r * L + l] - mx[r]);
  }
  sync;
  if (j == 0) {
    dn = 0;
    for (l = 0; l < L; l++) {
      dn += sc[r * L + l];
    }
    den[r] = dn;
  }
  sync;
  for (e = j; e < D; e += TPR) {
    acc = 0;
    for (l = 0; l < L; l++) {
      acc += sc[r * L + l] * vmat[l * D + e];
    }
    o[r * D + e] = acc / den[r];
  }
}
