import torch, time
torch.manual_seed(0)
for (m, k, n) in [(10000, 784, 60000), (4096, 784, 60000), (2048, 784, 60000), (10000, 128, 60000)]:
    a = torch.randint(-128, 127, (m, k), dtype=torch.int8, device='cuda')
    b = torch.randint(-128, 127, (n, k), dtype=torch.int8, device='cuda')
    for _ in range(3):
        c = torch._int_mm(a, b.t())
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        c = torch._int_mm(a, b.t())
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f'{m}x{k}x{n}: {ms:.3f} ms  {2*m*k*n/ms/1e9:.0f} TOPS  out {c.numel()*4/1e9:.2f} GB', flush=True)
# also check exactness against fp64
a = torch.randint(-128, 127, (64, 784), dtype=torch.int8, device='cuda')
b = torch.randint(-128, 127, (128, 784), dtype=torch.int8, device='cuda')
c = torch._int_mm(a, b.t()).cpu().long()
ref = (a.cpu().long() @ b.cpu().long().t())
print('exact', bool((c == ref).all()))
