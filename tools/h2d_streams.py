import torch, time
n = 64 * 1024 * 1024  # 256 MiB int32
h = torch.empty(n, dtype=torch.int32).pin_memory(); d = torch.empty(n, dtype=torch.int32, device="cuda")
s = [torch.cuda.Stream() for _ in range(4)]
def run(k):
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    e0.record(cur)
    for st in s[:k]: st.wait_event(e0)
    part = n // k
    for i, st in enumerate(s[:k]):
        with torch.cuda.stream(st):
            d[i*part:(i+1)*part].copy_(h[i*part:(i+1)*part], non_blocking=True)
    for st in s[:k]:
        ev = torch.cuda.Event(); ev.record(st); cur.wait_event(ev)
    e1.record(cur); torch.cuda.synchronize()
    return e0.elapsed_time(e1)
for k in (1, 2, 4, 1, 2, 4):
    t = min(run(k) for _ in range(5))
    print(k, "streams:", round(t, 3), "ms", round(n*4/t/1e6, 1), "GB/s")
