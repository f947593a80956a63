"""H2D copy rate of one step's fp32 ResNet-18 input (154 MB, pinned host memory) split over
1, 2 or 4 CUDA streams (the e2e bound): python tests/h2d_rate.py"""
import torch, time
n = 154140672 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
def run(k, reps=20):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for _ in range(reps):
        ev = []
        for i in range(k):
            st = s[i]
            st.wait_stream(cur)
            with torch.cuda.stream(st):
                a, b = i * n // k, (i + 1) * n // k
                d[a:b].copy_(h[a:b], non_blocking=True)
        for i in range(k): cur.wait_stream(s[i])
    e1.record(cur)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    return n * 4 / ms / 1e6
for k in (1, 2, 4, 1, 2, 4):
    print(k, "streams: %.1f GB/s" % run(k))
