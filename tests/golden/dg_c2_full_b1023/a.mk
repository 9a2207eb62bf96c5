// C2 reference: one thread folds its CTA's slice left to right.
kernel reduce_seq {
  param B;
  param BS;
  param N;
  in x[N];
  out y[1];

  s = 0;
  for (i = 0; i < BS; i++) {
    s += x[B * BS + i];
  }
  y[0] = s;
}
