import torch, time
n = 16_411_928 // 8
h = torch.empty(n, dtype=torch.int64).pin_memory()
d = torch.empty(n, dtype=torch.int64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=20):
    fn(); torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    a.record(); [fn() for _ in range(reps)]; b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / reps
print("1 copy  ms", t(lambda: d.copy_(h, non_blocking=True)))
def two():
    half = n // 2
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1): d[:half].copy_(h[:half], non_blocking=True)
    with torch.cuda.stream(s2): d[half:].copy_(h[half:], non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)
print("2 streams ms", t(two))
def chunks():
    q = n // 8
    for i in range(8): d[i*q:(i+1)*q].copy_(h[i*q:(i+1)*q], non_blocking=True)
print("8 chunks ms", t(chunks))
