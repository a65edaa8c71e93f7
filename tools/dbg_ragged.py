import sys; sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/tests')
import numpy as np, torch
from test_gpu_parity import *
sizes = [0, 1, 17, 4097, 65536 * 3 + 5, 0, 250_001, 2, 31, 33]
p = E.Params(torch.bfloat16, 3, 1e-3, 4)
Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 300 + i) for i, n in enumerate(sizes)]
Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 400 + i) for i, n in enumerate(sizes)]
C0s = [synth.quantile_centroids(8, 1.0) for _ in sizes]
gpu = run_gpu(Ws, Gs, C0s, p)
for t, n in enumerate(sizes):
    if n == 0: continue
    ref = oracle_dense(bits_of(Ws[t]), Gs[t].double().numpy(), C0s[t], p)
    print(n, "minS/n", np.min(ref["St"]) / n, "dC gpu", gpu["dC0"][t], "ref", ref["dC"])
