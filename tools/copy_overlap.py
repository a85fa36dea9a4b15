"""Do an H2D copy on one stream and a D2H copy on another overlap on this box?"""
import time, torch
d_out = torch.empty(24 << 20, dtype=torch.uint8, device="cuda")
h_out = torch.empty(24 << 20, dtype=torch.uint8, pin_memory=True)
h_in = torch.empty(4 << 20, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
for trial in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    ev[0].record(sa)
    with torch.cuda.stream(sa):
        h_out.copy_(d_out, non_blocking=True)
    ev[1].record(sa)
    ev[2].record(sb)
    with torch.cuda.stream(sb):
        d_in.copy_(h_in, non_blocking=True)
    ev[3].record(sb)
    torch.cuda.synchronize()
    print(f"d2h {ev[0].elapsed_time(ev[1]):.3f} ms; h2d starts at {ev[0].elapsed_time(ev[2]):.3f}, "
          f"ends at {ev[0].elapsed_time(ev[3]):.3f} ms")
