"""Host<->device copy bandwidth from pinned memory: H2D alone, D2H alone, both at once (two streams),
for chunk sizes as used by pipeline.HostPipeline.  python tools/pcie_bw.py"""
import torch

GB = 1 << 30
n = 4 * GB
h_in = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(n, dtype=torch.uint8, device="cuda")
d_out = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h, chunk):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    for o in range(0, n, chunk):
        if h2d:
            with torch.cuda.stream(s1):
                d_in[o:o + chunk].copy_(h_in[o:o + chunk], non_blocking=True)
        if d2h:
            with torch.cuda.stream(s2):
                h_out[o:o + chunk].copy_(d_out[o:o + chunk], non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return n / (e0.elapsed_time(e1) / 1e3) / 1e9


for chunk in (64 << 20, 256 << 20, 1 << 30):
    run(True, True, chunk)
    print(f"chunk {chunk >> 20:5d} MiB: H2D {run(True, False, chunk):6.1f} GB/s  D2H {run(False, True, chunk):6.1f} GB/s  "
          f"both {run(True, True, chunk):6.1f} GB/s each way")
