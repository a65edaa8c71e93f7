"""torchrun --nproc-per-node 1: CUDA-event timing of each piece of the page-compact count exchange
inside a loop like bench.py's, with the library comm (edkm.Comm) at nranks = 1."""
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
plan = E.Plan([w.numel() for w in Ws], p, dev)
s = torch.cuda.current_stream()
for it in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(8)]
    torch.cuda.synchronize()
    ev[0].record(s); plan.uniquify(Ws); ev[1].record(s)
    mask = plan.count_pages(); ev[2].record(s)
    comm.allreduce(mask, op=E.MAX); ev[3].record(s)
    th = time.perf_counter(); host = union_pages(mask); pages = host.to(dev); th = time.perf_counter() - th
    ev[4].record(s); comp = plan.pack_counts(pages); ev[5].record(s)
    comm.allreduce(comp); ev[6].record(s)
    plan.unpack_counts(pages, comp); ev[7].record(s)
    torch.cuda.synchronize()
    names = ["F1", "count_pages", "AR mask", "host gap", "pack", "AR compact", "unpack"]
    print({n: round(ev[i].elapsed_time(ev[i + 1]), 3) for i, n in enumerate(names)}, "host", round(th * 1e3, 3))
comm.close()
dist.destroy_process_group()
