#!/usr/bin/env python
"""eDKM hot-path benchmark: DKM fwd+bwd weights/sec on LLaMA-7B-shaped weights, 3-bit.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--workload cfg3] [--impl ours|reference]

One step = the whole hot path over every tensor of the workload (S1):
F1 uniquify -> [counts all-reduce] -> TF forward iterations -> F2 reconstruct (W~, bf16)
-> B1 buckets + gamma_T -> [gamma all-reduce] -> TB reverse loop + B2 dW (bf16).
N=1 runs BASELINE.json's metric configuration (configs[2], full LLaMA-7B: 226 tensors,
6,738,149,376 weights) on one B200; under torchrun the model is sharded by tensor (whole
tensors per rank, balanced longest-first: independent clustering problems, no data-path
exchange; EDKM_SHARD=slice: the contiguous slice of every tensor, with the count and
gamma all-reduces) -- total work fixed, so "scaling": "strong".
Prints ONE JSON line on rank 0.  Timing: W warm-up steps, then K steps bracketed by
barrier + synchronize, CUDA events on the launching stream, max over ranks.  Inputs
(27 GB of W and G per step) exceed the 126 MB L2, so no flush is needed.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "DKM fwd+bwd weights/sec (LLaMA-7B, 3-bit) at 1/2/4/8 B200; % HBM peak"
# algorithmic HBM bytes per weight of each per-weight pass (S4), bf16 I/O
BYTES_PER_WEIGHT = {"F1": 2, "F2": 4, "B1": 4, "B2": 6}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--e2e-groups", type=int, default=32)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="skip the CUDA-graph replay timing")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--no-clocks", action="store_true", help="no nvidia-smi sampling during the timed steps")
    return ap.parse_args()


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu --set full summary, or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_full_summary.json")) as f:
            d = json.load(f)
        return d["kernels"][kernel]["dram_bytes_per_weight"]
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region.  nvidia-smi writes to a
    file (no Python reader thread runs while the step is timed: a thread reading its pipe delayed
    the host's wake-up in the mid-step sync of the page-compact exchange, AR_counts 0.24 -> 1.2-1.6 ms)."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int, enabled: bool = True):
        self.index, self.proc, self.lines, self.enabled = index, None, [], enabled
        self.path = None

    def __enter__(self):
        if not self.enabled:
            return self
        try:
            import tempfile
            fd, self.path = tempfile.mkstemp(prefix="edkm_clk_", suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "50", "-f", self.path],
                                         stdout=subprocess.DEVNULL, stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.path:
            try:
                with open(self.path) as f:
                    self.lines = [ln.strip() for ln in f]
                os.unlink(self.path)
            except OSError:
                pass

    def summary(self):
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        sm, mx, reasons = [], 0.0, set()
        for ln in self.lines:
            parts = [x.strip() for x in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(n)
        sm.sort()
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": mx or None, "reasons": sorted(reasons),
                "samples": len(sm)}


# ----------------------------------------------------------------------------- reference arm (CPU oracle)
def oracle_sample_step(w_bits, G, C0, wl, nthreads):
    import numpy as np

    from oracle import oracle as O
    dt = O.BF16 if str(wl.wdtype).endswith("bfloat16") else O.FP16
    w = O.decode16(w_bits, dt)
    Ct, St, T = O.dkm_forward(w, np.float32(C0).astype(np.float64), wl.tau, wl.max_iter, nthreads=nthreads)
    Wt = O.reconstruct(w, Ct[-1], wl.tau)
    dW, dC = O.dkm_backward(w, G, Ct, St, wl.tau, nthreads=nthreads)
    return w.size, (Ct[-1], Wt, dW, dC)


def cpu_sample(wl, n_target, seed_t=1):
    """Bounded sample of the workload: the first n weights of tensor 1 (layer 0 q_proj), same law."""
    import numpy as np
    import torch

    from paper_2309_00964_b200 import synth
    n = min(n_target, wl.shapes[seed_t][1] * wl.shapes[seed_t][2])
    W = synth.weights(wl, seed_t, "cpu", n=n)
    G = synth.grads(wl, seed_t, "cpu", n=n)
    return (W.view(torch.int16).numpy().view(np.uint16), G.double().numpy(), synth.quantile_centroids(wl.k, wl.sigma))


def calibrate_cpu(wl, seconds, nthreads):
    n0 = 1 << 20
    b, G, C0 = cpu_sample(wl, n0)
    t0 = time.perf_counter()
    oracle_sample_step(b, G, C0, wl, nthreads)
    dt = time.perf_counter() - t0
    return max(n0, int(n0 * seconds / max(dt, 1e-6)))


def cpu_baseline(wl, seconds, gpu_result=None, fetch=None, tensors=None):
    """Dense oracle over whole tensors of layer 0 (q, k, v, ...) in order until ~`seconds` elapse, on
    every host core; then the same oracle on ONE thread over a 1M-weight sample.  `gpu_result(t)` gives
    the bench step's own outputs for tensor t (C_T, dC_0 and this rank's slice of W~, dW); they are
    compared with the oracle's outputs for the tensors timed here (untimed), as the line's parity.
    `fetch(t)` gives the bench's own (W bits, G) of the whole tensor t (else the same law on the CPU)."""
    import numpy as np
    cores = len(os.sched_getaffinity(0))
    done, names, refs, tt = 0, [], {}, 0.0
    for t in (range(1, len(wl.shapes)) if tensors is None else tensors):
        n = wl.shapes[t][1] * wl.shapes[t][2]
        b, G, C0 = cpu_sample(wl, n, seed_t=t)
        if fetch is not None:
            b, G = fetch(t)
        t0 = time.perf_counter()
        _, refs[t] = oracle_sample_step(b, G, C0, wl, cores)
        tt += time.perf_counter() - t0
        done += b.size
        names.append(wl.shapes[t][0])
        if tt >= seconds:
            break
    dt = tt
    b1, G1, C01 = cpu_sample(wl, 1 << 20, seed_t=1)
    t1 = time.perf_counter()
    oracle_sample_step(b1, G1, C01, wl, 1)
    dt1 = time.perf_counter() - t1
    out = {"value": done / dt, "unit": "weights/s", "cores": cores, "kind": "oracle",
           "sample": f"dense fp64 oracle fwd+bwd (all |W|x|C| entries, T={wl.max_iter}, k={wl.k}, tau={wl.tau}) "
                     f"on whole tensors {names} ({done} weights, {wl.name} law), {dt:.1f} s on {cores} threads",
           "value_1thread": b1.size / dt1,
           "sample_1thread": f"the same oracle on 1 thread, first {b1.size} weights of {wl.shapes[1][0]}, {dt1:.1f} s"}
    if gpu_result is not None:
        def nw(a, r):
            a, r = np.asarray(a, np.float64), np.asarray(r, np.float64)
            return float(np.max(np.abs(a - r)) / max(np.max(np.abs(r)), 1e-300)) if r.size else 0.0
        par = {"tensors": names, "C_T": 0.0, "dC0": 0.0, "W~": 0.0, "dW": 0.0}
        for t, (CT, Wt, dW, dC) in refs.items():
            g = gpu_result(t)
            lo, hi = g["slice"]
            par["C_T"] = max(par["C_T"], nw(g["C"], CT))
            par["dC0"] = max(par["dC0"], nw(g["dC0"], dC))
            # 16-bit outputs: normwise against the fp64 oracle (includes the bf16 rounding, ~2^-9)
            par["W~"] = max(par["W~"], nw(g["Wt"], Wt[lo:hi]))
            par["dW"] = max(par["dW"], nw(g["dW"], dW[lo:hi]))
        par["note"] = ("normwise max|x - x_ref| / max|x_ref| of the step's own outputs vs the dense oracle on the "
                       "tensors above; C_T, dC_0 fp32 (bar 1e-5), W~ and dW are the bf16/fp16 outputs (their "
                       "rounding, up to 2^-8 / 2^-11 relative, included)")
        out["parity"] = par
    return out


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2309_00964_b200 import synth
    wl = synth.workload(args.workload)
    cores = len(os.sched_getaffinity(0))
    n = calibrate_cpu(wl, 3.0, cores)
    b, G, C0 = cpu_sample(wl, n)
    for _ in range(args.warmup):
        oracle_sample_step(b, G, C0, wl, cores)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle_sample_step(b, G, C0, wl, cores)
    dt = (time.perf_counter() - t0) / max(args.steps, 1)
    v = b.size / dt
    sample = (f"each step: dense fp64 oracle fwd+bwd on the first {b.size} weights of {wl.shapes[1][0]} "
              f"({wl.name}: k={wl.k}, tau={wl.tau}, T={wl.max_iter})")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": v, "unit": "weights/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": f"{wl.name} (bounded sample)", "weights_per_step": int(b.size)},
        "cpu_baseline": {"value": v, "unit": "weights/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": v, "unit": "weights/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0}))


# ----------------------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    import torch
    import torch.distributed as dist

    from paper_2309_00964_b200 import build as B
    from paper_2309_00964_b200 import edkm as E
    from paper_2309_00964_b200 import synth
    from paper_2309_00964_b200.dist import assign_tensors, exchange_counts_compact, shard_range

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    launched = "RANK" in os.environ and "MASTER_ADDR" in os.environ  # under torchrun: always use the process group
    distributed = world > 1 or launched
    # EDKM_DIST_BACKEND=gloo: a check of the multi-rank orchestration with every rank on the GPUs
    # there are (e.g. two ranks sharing one B200); the bench itself uses NCCL, one rank per GPU
    backend = os.environ.get("EDKM_DIST_BACKEND", "nccl")
    if distributed and backend != "nccl":
        local = local % torch.cuda.device_count()
    if distributed:
        torch.cuda.set_device(local)
        if backend == "nccl":
            # NCCL's init lines (rank, nRanks, transports) stay visible on stderr at N > 1
            # (the image presets NCCL_DEBUG=VERSION, whose one line NCCL writes to stdout; at INFO it
            # honours NCCL_DEBUG_FILE, so the version and INIT lines go to stderr and stdout keeps the
            # one JSON line)
            if os.environ.get("NCCL_DEBUG", "").upper() in ("", "VERSION", "WARN"):
                os.environ["NCCL_DEBUG"] = "INFO"
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    if rank == 0:
        B.build()
    if distributed:
        dist.barrier()
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    wl = synth.workload(args.workload)
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter, wl.eps)

    # ---- synthetic inputs, resident in HBM (this rank's whole tensors, or its slice of every tensor)
    # Sharding at N > 1 (EDKM_SHARD): "tensor" (default while the largest tensor fits a rank's share):
    # whole tensors per rank (dist.assign_tensors, longest-first greedy), independent clustering
    # problems (one C per tensor, R12), so the step has no data-path exchange and no replicated table
    # phase; "slice": the contiguous slice of every tensor with the count and gamma all-reduces.
    all_n = [r * c for _, r, c in wl.shapes]
    smode = os.environ.get("EDKM_SHARD", "auto")
    if smode == "auto":
        smode = "tensor" if world > 1 and max(all_n) <= sum(all_n) / world else "slice"
    tensor_mode = smode == "tensor"
    owned = assign_tensors(all_n, world)[rank] if tensor_mode else list(range(len(all_n)))
    Ws, Gs, numels = [], [], []
    for t in owned:
        lo, hi = (0, all_n[t]) if tensor_mode else shard_range(all_n[t], rank, world)
        w = synth.weights(wl, t, dev)[lo:hi].contiguous()
        g = synth.grads(wl, t, dev)[lo:hi].contiguous()
        Ws.append(w)
        Gs.append(g)
        numels.append(hi - lo)
    n_local = sum(numels)
    n_total = wl.numel
    # N > 1: split the table phase by tensor block when it is heavy (k T >= 64, e.g. CFG4's k=16, T=30):
    # each rank runs TF/TB for its block and derives the other tensors' layout from the global counts;
    # the ranks exchange the owners' states, trajectories and the populated pages of their tables
    # (dist.ShardedStep(compact_tables=True)).  CFG3 (k T = 40) stays replicated by default: at N = 8
    # the estimated split (own block TF + TB ~0.18 ms, layout pass ~0.03, five all-gathers ~0.1) saves
    # ~0.04 ms of ~0.38; EDKM_SHARD_TABLE=1 forces the split, 0 disables it.
    tmode = os.environ.get("EDKM_SHARD_TABLE", "auto")
    shard = not tensor_mode and (tmode == "1" or (world > 1 and tmode == "auto" and wl.k * wl.max_iter >= 64))
    if shard:
        from paper_2309_00964_b200.dist import allgather_blocks, padded_numels
        npad = len(padded_numels(numels, world)) - len(numels)
        Ws += [torch.empty(0, dtype=wl.wdtype, device=dev)] * npad
        Gs += [torch.empty(0, dtype=wl.wdtype, device=dev)] * npad
        numels += [0] * npad
        blk = len(numels) // world
        t0, t1 = rank * blk, (rank + 1) * blk
    C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
    Wt = [torch.empty_like(w) for w in Ws]
    dW = [torch.empty_like(w) for w in Ws]
    plan = E.Plan(numels, p, dev)
    views = plan.views() if shard else None
    stream = torch.cuda.current_stream()

    # N > 1 collectives: by default on libedkm.so's own NCCL communicator (edkm.Comm, SURVEY S8(b):
    # edkm_comm_allreduce / _allgather on the step's stream); EDKM_COMM=torch uses torch.distributed
    comm = None  # (by tensor there is no data-path collective: torch.distributed times the step)
    if distributed and backend == "nccl" and not tensor_mode and os.environ.get("EDKM_COMM", "lib") == "lib":
        try:
            comm = E.Comm()
        except Exception as e:  # every rank fails alike (same library, same NCCL): torch's NCCL instead
            print(f"bench: libedkm.so NCCL comm unavailable ({e}); collectives via torch.distributed",
                  file=sys.stderr)
            comm = None

    def allreduce(t, op=None):
        op = dist.ReduceOp.SUM if op is None else op
        if not distributed:
            return
        if comm is not None:
            comm.allreduce(t, op=E.MAX if op == dist.ReduceOp.MAX else E.SUM)
        elif backend == "nccl":
            dist.all_reduce(t, op=op)
        else:  # gloo check mode: through host memory
            h = t.cpu()
            dist.all_reduce(h, op=op)
            t.copy_(h)

    def allreduce_max(t):
        allreduce(t, op=dist.ReduceOp.MAX)

    def allgather(full):
        if comm is not None:
            return comm.allgather_blocks(full)
        if backend == "nccl":
            return allgather_blocks(full)
        P = dist.get_world_size()  # gloo check mode: rank blocks through host memory
        b = full.shape[0] // P
        parts = [torch.empty_like(full[:b], device="cpu") for _ in range(P)]
        dist.all_gather(parts, full[rank * b:(rank + 1) * b].cpu())
        full.copy_(torch.cat(parts))
        return full

    # N > 1: exchange 1 fused into F1 over NVLS (dist.NvlsCounts) when the system supports it and
    # it passes a bit-exact self-check against F1 + NCCL all-reduce; otherwise NCCL.
    # exchange 1: the whole int32 counts by default.  EDKM_COMPACT=1: only the populated 256-pattern
    # pages (dist.exchange_counts_compact; also the compact table split) -- it needs
    # one mid-step host read of the page mask, and that sync measured 0.24 ms alone but ~1-1.6 ms per
    # step while nvidia-smi samples the clocks (bench at N=1 under torchrun), more than the ~0.1 ms
    # it can save on a 59 MB NVLink all-reduce at N = 8
    compact = distributed and not tensor_mode and os.environ.get("EDKM_COMPACT", "0") == "1"
    via = "libedkm.so's NCCL comm (edkm_comm_*)" if comm is not None else f"torch.distributed ({backend})"
    nv, exchange = None, (f"counts: {'page-compact ' if compact else ''}int32 all-reduce; gamma: fp64 all-reduce; "
                          f"via {via}")
    if tensor_mode:
        exchange = ("none: each rank clusters whole tensors (independent problems, one C per tensor, R12); "
                    f"only the step time's max over ranks crosses them (via {via})")
    # the NVLS-fused count exchange (multimem reductions inside F1) has not yet run on NVSwitch
    # hardware: opt-in (EDKM_NVLS=1) until it has been validated there
    mode = os.environ.get("EDKM_NVLS", "0")
    if not tensor_mode and ((world > 1 and mode != "0") or mode == "emulate"):  # emulate: plain memory, one rank
        from paper_2309_00964_b200.dist import NvlsCounts
        try:
            nv = NvlsCounts(len(Ws), dev, emulate=mode == "emulate")
            # the first exchange may not trap on a timeout (multicast set up but not delivering):
            # it records the failure and the check below falls back to NCCL on every rank
            E.nvls_set_timeout(10.0, trap=False)
            got = plan.uniquify_nvls(Ws, nv).clone()
            timed_out = E.nvls_failed()
            E.nvls_set_timeout(20.0, trap=True)
            want = E.uniquify(Ws, p)
            allreduce(want)
            ok = torch.tensor([float(not timed_out and torch.equal(got, want))], device=dev)
            if distributed:
                allreduce(ok, op=dist.ReduceOp.MIN)
            if ok.item() != 1.0:
                raise RuntimeError("NVLS counts differ from the NCCL all-reduce")
            exchange = "counts: NVLS multimem reductions fused into F1 + in-kernel arrival barrier; gamma: nccl all-reduce"
            if rank == 0:
                print(f"bench: NVLS count exchange self-check passed ({'emulate' if mode == 'emulate' else 'multicast'})",
                      file=sys.stderr)
        except Exception as e:  # no multicast, or a failed self-check: NCCL
            if rank == 0:
                print(f"bench: NVLS count exchange unavailable ({e}); using NCCL", file=sys.stderr)
            nv = None
            plan.counts = torch.empty((plan.nt, E.PATTERNS), dtype=torch.int32, device=dev)

    from paper_2309_00964_b200.dist import ShardedStep
    # the page-exchange helper of the compact table split (the step below drives the calls itself so
    # that it can record events between them)
    ss = ShardedStep(plan, allreduce=lambda t: allreduce(t), allgather=lambda t: allgather(t),
                     allreduce_max=allreduce_max, shard_table=shard, compact_tables=shard and compact)

    def step(ev=None):
        # the seven kernels of the hot path, one C-ABI call each, events between them
        def mark(i):
            if ev is not None:
                ev[i].record(stream)
        mark(0)
        if nv is not None:
            plan.uniquify_nvls(Ws, nv)       # F1 + exchange 1 in the NVSwitch (N > 1)
            mark(1)
        else:
            plan.uniquify(Ws)                # F1
            mark(1)
            if compact:                      # exchange 1 (N > 1), populated pages only
                ss.page_list = exchange_counts_compact(plan, allreduce, allreduce_max)
            elif not tensor_mode:
                allreduce(plan.counts)       # exchange 1 (N > 1, slices)
        mark(2)
        if shard:
            plan.forward_range(t0, t1, C0)   # TF, this rank's tensor block
            if compact and nv is None:       # others: layout locally, owners' states + populated pages
                if t0 > 0:
                    plan.forward_layout_range(0, t0)
                if t1 < plan.nt:
                    plan.forward_layout_range(t1, plan.nt)
                for name in ("state", "ctraj", "C_out"):
                    allgather(views[name])
                ss._exchange_pages("table16")
            else:
                for name in ("state", "ctraj", "rows", "page_cnt", "C_out", "table16"):
                    allgather(views[name])
        else:
            plan.forward(C0)                 # TF
        mark(3)
        plan.reconstruct(Ws, Wt, E.SOFT)     # F2
        mark(4)
        plan.backward_buckets(Ws, Gs)        # B1
        mark(5)
        plan.backward_gamma()                # TGAMMA
        mark(6)
        if not tensor_mode:
            allreduce(plan.gamma)            # exchange 2 (N > 1, slices)
        mark(7)
        if shard:
            plan.backward_table_range(t0, t1)  # TB, this rank's tensor block
            if compact and nv is None:
                ss._exchange_pages("phipsi")
                allgather(views["dC0"])
            else:
                for name in ("phipsi", "dC0"):
                    allgather(views[name])
        else:
            plan.backward_table()            # TB
        mark(8)
        plan.backward_dw(Ws, Gs, dW)         # B2
        mark(9)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # per-phase events in every timed step (same stream as the kernels)
    evs = [[torch.cuda.Event(enable_timing=True) for _ in range(10)] for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if distributed:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local, enabled=not args.no_clocks) as clk:
        start.record(stream)
        for s in range(args.steps):
            step(evs[s])
        stop.record(stream)
        torch.cuda.synchronize()
    if distributed:
        dist.barrier()
    ms = start.elapsed_time(stop) / args.steps
    names = ["F1", "AR_counts", "TF", "F2", "B1", "TGAMMA", "AR_gamma", "TB", "B2"]
    phase = {n: sum(evs[s][i].elapsed_time(evs[s][i + 1]) for s in range(args.steps)) / args.steps
             for i, n in enumerate(names)}
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if distributed:
        allreduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    launches_per_step = 7 + (nv is not None) + 3 * (compact and nv is None)  # + NVLS barrier / page exchange
    if shard and compact and nv is None:  # TF layout passes + page packs / unpacks of table16 and (phi, psi)
        lists = ss._pg_cache["lists"][1]
        launches_per_step += int(t0 > 0) + int(t1 < plan.nt) + 2 * sum(1 for x in lists if x.numel())
    # N > 1: C_T and dC_0 must be bit-identical on every rank ("weights are identical in each
    # learner"): all-gather a hash of their bytes and fail on any mismatch
    rank_identical = None
    if distributed and not tensor_mode:  # (by tensor, every C_T / dC_0 is computed on one rank only)
        import hashlib
        hsh = hashlib.sha256(plan.C_out.cpu().numpy().tobytes() + plan.dC0.cpu().numpy().tobytes()).digest()[:8]
        mine = torch.tensor([int.from_bytes(hsh, "little", signed=True)], dtype=torch.int64)
        allh = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        if backend == "nccl":
            got = torch.zeros(world, dtype=torch.int64, device=dev)
            dist.all_gather_into_tensor(got, mine.to(dev))
            allh = got.cpu().tolist()
        else:
            dist.all_gather(allh, mine)
            allh = [int(x.item()) for x in allh]
        rank_identical = len(set(allh)) == 1
        if not rank_identical:
            raise RuntimeError(f"C_T / dC_0 differ across ranks (hashes {allh})")

    # ---- the same step captured once as a CUDA graph and replayed (Plan.graph; one GPU)
    graph = None
    if not distributed and not args.no_graph:
        g = plan.graph(Ws, Gs, C0, Wt, dW)
        for _ in range(args.warmup):
            g.replay()
        torch.cuda.synchronize()
        g0, g1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g0.record(stream)
        for _ in range(args.steps):
            g.replay()
        g1.record(stream)
        torch.cuda.synchronize()
        gms = g0.elapsed_time(g1) / args.steps
        graph = {"ms_per_step": gms, "value": n_total / (gms / 1e3), "unit": "weights/s",
                 "note": "Plan.graph: memsets + 7 kernels captured once, replayed (no per-phase events)"}
        del g

    # ---- end to end through the public API with host buffers (H2D of W, G; D2H of W~, dW every step)
    e2e = None
    if not args.no_e2e:
        hW = [torch.empty(w.shape, dtype=w.dtype, pin_memory=True) for w in Ws]
        hG = [torch.empty(g.shape, dtype=g.dtype, pin_memory=True) for g in Gs]
        hWt = [torch.empty(w.shape, dtype=w.dtype, pin_memory=True) for w in Ws]
        hdW = [torch.empty(w.shape, dtype=w.dtype, pin_memory=True) for w in Ws]
        for a, b in zip(hW, Ws):
            a.copy_(b)
        for a, b in zip(hG, Gs):
            a.copy_(b)
        torch.cuda.synchronize()

        from paper_2309_00964_b200.pipeline import HostPipeline
        pipe = HostPipeline(numels, p, dev, n_groups=args.e2e_groups,
                            allreduce=allreduce if distributed and not tensor_mode else None,
                            buffers=(Ws, Gs, Wt, dW))

        def e2e_step():
            pipe.step(hW, hG, C0, hWt, hdW)

        e2e_step()
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.e2e_steps):
            e2e_step()
        e1.record(stream)
        torch.cuda.synchronize()
        te = torch.tensor([e0.elapsed_time(e1) / args.e2e_steps], dtype=torch.float64, device=dev)
        if distributed:
            allreduce(te, op=dist.ReduceOp.MAX)
        # whole-job bytes (every rank copies its own slices)
        nb = torch.tensor([sum(w.numel() * 2 + g.numel() * 2 for w, g in zip(Ws, Gs)),
                           sum(w.numel() * 2 * 2 for w in Ws)], dtype=torch.float64, device=dev)
        allreduce(nb)
        bytes_in, bytes_out = int(nb[0].item()), int(nb[1].item())
        e2e = {"value": n_total / (float(te.item()) / 1e3), "unit": "weights/s", "h2d_bytes_per_step": bytes_in,
               "d2h_bytes_per_step": bytes_out, "ms_per_step": float(te.item()), "steps": args.e2e_steps,
               "path": f"pipeline.HostPipeline ({args.e2e_groups} tensor groups; H2D, the C-ABI step and D2H overlap on 3 streams); pinned host W, G in and W~, dW out every step"}
        del hW, hG, hWt, hdW

    if rank != 0:
        if comm is not None:
            comm.close()
        if distributed:
            dist.destroy_process_group()
        return

    w16 = "bf16" if wl.wdtype == torch.bfloat16 else "fp16"
    # ---- roofline of the dominant per-weight kernel (measured live above)
    peak, peak_src = measured_peaks()
    per_kernel = {k: phase[k] for k in ("F1", "F2", "B1", "B2")}
    dom = max(per_kernel, key=per_kernel.get)
    key = dom
    alg = BYTES_PER_WEIGHT[key] * n_local
    achieved = alg / (per_kernel[dom] / 1e3) / 1e9
    tr = ncu_traffic(key)
    roof = {"bound": "hbm", "kernel": key, "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": (tr * n_local if tr is not None else None),
            "traffic_source": "not measured in this run: dram__bytes_read.sum + dram__bytes_write.sum per weight of "
                              "this kernel from the committed ncu --set full capture (profiles/ncu_full_summary.json) "
                              "x the weights of one launch",
            "peak_source": peak_src, "algorithmic_bytes_per_launch": alg,
            "frac_of_spec_8tbs": achieved / 8000.0,
            "step_frac": (16 * n_local / (ms_max / 1e3) / 1e9) / peak,
            "step_frac_of_spec_8tbs": (16 * n_local / (ms_max / 1e3) / 1e9) / 8000.0}
    # ---- roofline of the table phase (TF + TGAMMA + TB): one ex2 per attention entry is the method's
    # irreducible transcendental work (U rows x k centroids per forward iteration, per reverse
    # iteration, and once each for the W~ table, gamma_T and the (phi, psi) table), counted from the
    # populated rows and the iterations each tensor ran; the peak is the MUFU ex2 rate measured on a
    # B200 (tools/ubench_mufu.cu, profiles/ubench_mufu_r02.txt: 15.97 ex2/clk/SM) at this run's
    # median SM clock.  The per-row arithmetic is fp32 FFMA/FADD around it (DESIGN S4), so the
    # kernels are issue-bound below this figure.
    tb0, tb1 = (t0, t1) if shard else (0, plan.nt)
    _, iters = E.read_status(plan.saved, plan.nt, p)
    rows_t = (plan.counts[tb0:tb1] != 0).sum(dim=1).tolist()
    ex2 = sum(u * wl.k * (2 * it + 3) for u, it in zip(rows_t, iters[tb0:tb1]))
    t_table = phase["TF"] + phase["TGAMMA"] + phase["TB"]
    sm_mhz = (clk.summary() or {}).get("sm_mhz") or 1965.0
    ex2_peak = 15.97 * torch.cuda.get_device_properties(dev).multi_processor_count * sm_mhz * 1e6
    table_roof = {"bound": "xu", "op": "ex2.approx.ftz.f32 (one per attention entry)", "kernels": "TF+TGAMMA+TB",
                  "rows": int(sum(rows_t)), "ex2_per_step": int(ex2), "ms": t_table,
                  "achieved": ex2 / (t_table / 1e3), "peak": ex2_peak, "unit": "ex2/s",
                  "frac": ex2 / (t_table / 1e3) / ex2_peak,
                  "peak_source": f"measured 15.97 ex2/clk/SM (tools/ubench_mufu.cu) x SMs x {sm_mhz:.0f} MHz"}
    out = {
        "metric": METRIC, "value": n_total / (ms_max / 1e3), "unit": "weights/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": w16, "data": "synthetic",
        "config": {"workload": f"{wl.name}: LLaMA-7B-shaped, {len(wl.shapes)} tensors, {n_total} weights, "
                               f"{'bf16' if wl.wdtype == torch.bfloat16 else 'fp16'} N(0,{wl.sigma}^2), "
                               f"b={wl.bits} (k={wl.k}), tau={wl.tau}, T={wl.max_iter}",
                   "tensors": len(wl.shapes), "weights": n_total, "bits": wl.bits, "tau": wl.tau,
                   "iters": wl.max_iter, "parallelism": f"{'tensors' if tensor_mode else 'slices'}{world}",
                   "exchange": exchange,
                   "table_phase": ("this rank's own tensors only" if tensor_mode and world > 1 else
                                   "split by tensor block + " + ("page-compact exchange" if compact and nv is None
                                                                 else "all-gather") if shard
                                   else "replicated on every rank"),
                   "rank_weights": ([sum(all_n[t] for t in o) for o in assign_tensors(all_n, world)]
                                    if tensor_mode and world > 1 else None),
                   "arith": f"{w16} I/O; exact integer F1/B1 sums, fp32 B2 FMA; table phase: fp32 per row "
                            "(ex2.approx), fp64 sums over rows, centroids and trajectories",
                   "l2": "no flush: 27 GB of W and G per step >> 126 MB L2"},
        "phases_ms": phase, "gpu_launches": launches_per_step * args.steps, "rank_identical_C_dC0": rank_identical,
        "clocks": clk.summary(), "roofline": roof, "table_roofline": table_roof, "e2e": e2e, "cuda_graph": graph,
    }
    if not args.no_cpu_baseline:  # rank 0 (at N > 1 too): the oracle on the host cores + the step's parity
        def gpu_result(t):  # t: the global tensor index; i: its index in this rank's plan
            i = owned.index(t)
            lo, hi = (0, all_n[t]) if tensor_mode else shard_range(all_n[t], rank, world)
            return {"C": plan.C_out[i].cpu().numpy(), "dC0": plan.dC0[i].cpu().numpy(), "slice": (lo, hi),
                    "Wt": Wt[i].double().cpu().numpy(), "dW": dW[i].double().cpu().numpy()}
        def fetch(t):  # the bench's own data of tensor t, whole (CUDA generator, as above)
            import numpy as np
            return (synth.weights(wl, t, dev).cpu().view(torch.int16).numpy().view(np.uint16),
                    synth.grads(wl, t, dev).double().cpu().numpy())
        # the oracle's tensors: layer 0 onwards (as at N = 1), or rank 0's own tensors by size when by tensor
        order = (sorted((t for t in owned if t > 0), key=lambda t: (all_n[t], t)) if tensor_mode and world > 1
                 else range(1, len(wl.shapes)))
        out["cpu_baseline"] = cpu_baseline(wl, args.cpu_seconds, gpu_result, fetch, tensors=order)
    print(json.dumps(out))
    if comm is not None:
        comm.close()
    if distributed:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
