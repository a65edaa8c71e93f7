"""Debug: run the bench step at N=2 (gloo check mode, both ranks on one GPU) and compare counts,
gamma, C_out, dC0 across ranks.  torchrun --nproc-per-node 2 tools/dbg_rank_identical.py cfg2 [compact]"""
import os, sys
import torch, torch.distributed as dist
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2309_00964_b200 import edkm as E, synth
from paper_2309_00964_b200.dist import shard_range, exchange_counts_compact

dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
dev = torch.device("cuda", 0)
wl = synth.workload(sys.argv[1])
compact = len(sys.argv) > 2 and sys.argv[2] == "compact"
p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
Ws, Gs = [], []
for t, (_, r, c) in enumerate(wl.shapes):
    lo, hi = shard_range(r * c, rank, world)
    Ws.append(synth.weights(wl, t, dev)[lo:hi].contiguous()); Gs.append(synth.grads(wl, t, dev)[lo:hi].contiguous())
plan = E.Plan([w.numel() for w in Ws], p, dev)
C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
Wt = [torch.empty_like(w) for w in Ws]; dW = [torch.empty_like(w) for w in Ws]
def ar(t, op=dist.ReduceOp.SUM):
    h = t.cpu(); dist.all_reduce(h, op=op); t.copy_(h)
for step in range(int(os.environ.get("STEPS", "1"))):
    plan.uniquify(Ws)
    if compact:
        exchange_counts_compact(plan, ar, lambda t: ar(t, dist.ReduceOp.MAX))
    else:
        ar(plan.counts)
    plan.forward(C0); plan.reconstruct(Ws, Wt); plan.backward_buckets(Ws, Gs); plan.backward_gamma()
    g_local = plan.gamma.clone()
    ar(plan.gamma)
    plan.backward_table(); plan.backward_dw(Ws, Gs, dW)
    torch.cuda.synchronize()
    res = {k: v.cpu() for k, v in dict(counts=plan.counts, C=plan.C_out, gamma=plan.gamma, dC0=plan.dC0).items()}
    out = [None] * world
    dist.all_gather_object(out, res)
    if rank == 0:
        for k in res:
            a, b = out[0][k], out[1][k]
            eq = torch.equal(a, b)
            print(step, k, "identical" if eq else f"DIFFER: {int((a != b).sum())} entries, max abs {float((a.double() - b.double()).abs().max())}")
dist.destroy_process_group()
