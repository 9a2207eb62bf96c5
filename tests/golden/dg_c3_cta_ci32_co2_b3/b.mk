// C3 candidate: im2col. Each thread stages its pixel's 3x3xCI patch as a
// column of the shared patch matrix, a barrier, then a K = 9*CI GEMM
// against the filter rows.
kernel conv_im2col {
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
  for (k = 0; k < CI * 9; k++) {
    col[k * TH * TW + tid] = x[((k / 9) * (H + 2) + oh + (k % 9) / 3) * (W + 2) + ow + k % 3];
  }
  sync;
  for (co = 0; co < CO; co++) {
    acc = 0;
    for (k = 0; k < CI * 9; k++) {
      acc += wt[co * CI * 9 + k] * col[k * TH * TW + tid];
    }
    y[co * TH * TW + tid] = acc;
  }
}
