// C3 reference: direct 3x3 convolution, one thread per output pixel.
kernel conv_direct {
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

  let oh = (B / TWS) * TH + tid / TW;
  let ow = (B % TWS) * TW + tid % TW;
  for (co = 0; co < CO; co++) {
    s = 0;
    for (ci = 0; ci < CI; ci++) {
      for (kh = 0; kh < 3; kh++) {
        for (kw = 0; kw < 3; kw++) {
          s += x[(ci * (H + 2) + oh + kh) * (W + 2) + ow + kw] * wt[(co * CI + ci) * 9 + kh * 3 + kw];
        }
      }
    }
    y[co * TH * TW + tid] = s;
  }
}
