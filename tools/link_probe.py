"""Host link probe: pinned H2D alone, D2H alone, and both at once on separate
streams (the e2e loop's traffic pattern).  Prints one JSON line (GB/s)."""
import json
import torch

def run(nb_h2d, nb_d2h, reps=20):
    dev = torch.device("cuda:0")
    hi = torch.empty(nb_h2d, dtype=torch.uint8).pin_memory() if nb_h2d else None
    di = torch.empty(nb_h2d, dtype=torch.uint8, device=dev) if nb_h2d else None
    ho = torch.empty(nb_d2h, dtype=torch.uint8).pin_memory() if nb_d2h else None
    do = torch.empty(nb_d2h, dtype=torch.uint8, device=dev) if nb_d2h else None
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    for _ in range(3):
        if hi is not None: di.copy_(hi, non_blocking=True)
        if ho is not None: ho.copy_(do, non_blocking=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_stream(torch.cuda.current_stream()); s2.wait_stream(torch.cuda.current_stream())
    for _ in range(reps):
        if hi is not None:
            with torch.cuda.stream(s1): di.copy_(hi, non_blocking=True)
        if ho is not None:
            with torch.cuda.stream(s2): ho.copy_(do, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    return reps * (nb_h2d + nb_d2h) / t / 1e9

h2d, d2h = 51609600, 18432048   # the c2 e2e step's bytes (bench.py)
print(json.dumps({"h2d_only_gbs": run(h2d, 0), "d2h_only_gbs": run(0, d2h), "both_total_gbs": run(h2d, d2h),
                  "both_ms_per_step": (h2d + d2h) / run(h2d, d2h) / 1e6}))
