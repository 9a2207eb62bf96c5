// C4 candidate: online softmax over key blocks of BC rows.
kernel attn_online {
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
  for (kb = 0; kb < L / BC; kb++) {
    for (l = j; l < BC; l += TPR) {
      acc = 0;
      for (e = 0; e < D; e++) {
        acc += q[qr * D + e] * kmat[(kb * BC + l) * D + e];
      }
      sb[r * BC + l] = acc;
    }
    sync;
    if (j == 0) {
      if (kb == 0) {
        m = NEG_INF;
      } else {
        m = ms[r];
      }
      mn = m;
      for (l = 0; l < BC; l++) {
        mn = max(mn, sb[r * BC + l]);
      }
      if (kb == 0) {
        dn = 0;
      } else {
        c = exp(m - mn);
        cs[r] = c;
        dn = ds[r] * c;
      }
      for (l = 0; l < BC; l++) {
        pl = exp(sb[r * BC + l] - mn);
        sb[r * BC + l] = pl;
        dn += pl;
      }
      ms[r] = mn;
      ds[r] = dn;
    }
    sync;
    for (e = j; e < D; e += TPR) {
      if (kb == 0) {
        acc = 0;
      } else {
        acc = oa[r * D + e] * cs[r];
      }
      for (l = 0; l < BC; l++) {
        acc += sb[r * BC + l] * vmat[(kb * BC + l) * D + e];
      }
      oa[r * D + e] = acc;
    }
    sync;
  }
  for (e = j; e < D; e += TPR) {
    o[r * D + e] = oa[r * D + e] / ds[r];
  }
}
