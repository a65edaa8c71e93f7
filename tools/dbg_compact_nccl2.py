"""torchrun --nproc-per-node 1: the full bench step with CUDA events around each piece of the
page-compact count exchange (library comm at nranks = 1)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, torch.distributed as dist
from paper_2309_00964_b200 import edkm as E, synth
from paper_2309_00964_b200.dist import union_pages

torch.cuda.set_device(0)
dist.init_process_group("nccl", device_id=torch.device("cuda", 0))
comm = E.Comm()
wl = synth.workload("cfg3")
dev = torch.device("cuda")
p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
Ws = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
Gs = [synth.grads(wl, t, dev) for t in range(len(wl.shapes))]
C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
Wt = [torch.empty_like(w) for w in Ws]; dW = [torch.empty_like(w) for w in Ws]
plan = E.Plan([w.numel() for w in Ws], p, dev)
s = torch.cuda.current_stream()
for it in range(6):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(9)]
    ev[0].record(s); plan.uniquify(Ws); ev[1].record(s)
    mask = plan.count_pages(); ev[2].record(s)
    comm.allreduce(mask, op=E.MAX); ev[3].record(s)
    host = union_pages(mask); ev[4].record(s)
    pages = host.to(dev); ev[5].record(s)
    comp = plan.pack_counts(pages); ev[6].record(s)
    comm.allreduce(comp); ev[7].record(s)
    plan.unpack_counts(pages, comp); ev[8].record(s)
    plan.forward(C0); plan.reconstruct(Ws, Wt); plan.backward_reduce(Ws, Gs, comm=comm); plan.backward_apply(Ws, Gs, dW)
    if it >= 2:
        torch.cuda.synchronize()
        names = ["F1", "count_pages", "AR mask", "D2H+host", "H2D", "pack", "AR compact", "unpack"]
        print({n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)})
comm.close()
dist.destroy_process_group()
