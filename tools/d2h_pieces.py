import time, torch
N = 18 << 20
K = 14
d = [torch.empty(N, dtype=torch.uint8, device="cuda") for _ in range(3)]
h = [torch.empty(N, dtype=torch.uint8, pin_memory=True) for _ in range(6)]
ss = [torch.cuda.Stream() for _ in range(3)]
for parts in (1, 4):
    for nstreams in (1, 3):
        best = 1e9
        for _ in range(5):
            torch.cuda.synchronize(); t0 = time.perf_counter()
            for k in range(K):
                s = ss[k % nstreams]
                with torch.cuda.stream(s):
                    for p in range(parts):
                        n = N // parts
                        h[k % 6][p*n:(p+1)*n].copy_(d[k % 3][p*n:(p+1)*n], non_blocking=True)
            torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
        print(f"parts {parts} streams {nstreams}: {K*N/best/1e9:.1f} GB/s")
