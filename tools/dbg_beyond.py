"""Diagnostic: the rows-beyond-the-stage parity case with every row staged (few tensors, cl = 8)
vs beyond the stage (38 tensors), same tensor 0, to separate a path error from conditioning."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np, torch
from paper_2309_00964_b200 import edkm as E, synth
import test_gpu_parity as T

for tau, c0kind in [(1.0, "data")]:
    for nt in (4, 38):
        rng = np.random.default_rng(7)
        Ws = []
        for i in range(nt):
            x = np.exp2(rng.uniform(-40, 12, 60_000)) * np.where(rng.random(60_000) < 0.5, -1.0, 1.0)
            Ws.append(torch.from_numpy(x).to(torch.bfloat16))
        Gs = [synth.normal_tensor(60_000, 1e-3, torch.bfloat16, 900 + i) for i in range(nt)]
        C0s = [synth.data_quantile_centroids(w, 8) if c0kind == "data" else synth.quantile_centroids(8, 2.0) for w in Ws]
        p = E.Params(torch.bfloat16, 3, tau, 3)
        gpu = T.run_gpu(Ws, Gs, C0s, p)
        wb = T.bits_of(Ws[0])
        ref = T.oracle_dense(wb, Gs[0].double().numpy(), C0s[0], p)
        e = {"C_T": T.normwise(gpu["C"][0], ref["Ct"][-1]), "dC0": T.normwise(gpu["dC0"][0], ref["dC"])}
        print(f"tau={tau} C0={c0kind} nt={nt}: {e}  C_T={np.round(ref['Ct'][-1], 4)}")
