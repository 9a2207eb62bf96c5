import sys, time
sys.path.insert(0, '/root/repo')
import torch
from paper_2511_12638_b200 import workloads, native as N
from paper_2511_12638_b200.engine import Session
w = workloads.c3_conv(64, 64, 256, 256, 16, 16)
for nodes in (1 << 22, 60_000_000):
    s = Session(0, max_nodes=nodes, max_kid_words=1 << 24, scratch_bytes=1 << 30)
    s.declare_inputs([("x", 64 * 258 * 258), ("wt", 64 * 64 * 9)])
    L = N.lib()
    for k in range(4):
        torch.cuda.synchronize(); t = time.perf_counter()
        L.veq_clear_terms(s.ctx); torch.cuda.synchronize()
        print(nodes, k, "clear %.2f ms" % (1000 * (time.perf_counter() - t)), flush=True)
    s.close()
