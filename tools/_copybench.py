import torch, time
a=torch.empty(4100,dtype=torch.float32,pin_memory=True); d=torch.empty(4100,device='cuda')
big=torch.empty(1215246,dtype=torch.int32,device='cuda'); big2=torch.empty_like(big)
torch.cuda.synchronize()
for name,f in [("h2d16k",lambda: d.copy_(a,non_blocking=True)),("d2h16k",lambda: a.copy_(d,non_blocking=True)),("d2d4.8M",lambda: big2.copy_(big)),("empty",lambda: torch.empty(1215246,dtype=torch.int32,device='cuda')),("event",lambda: torch.cuda.Event().record())]:
    for i in range(50): f()
    torch.cuda.synchronize()
    t=time.perf_counter()
    for i in range(200): f()
    t=time.perf_counter()-t
    torch.cuda.synchronize()
    print(name, f"{t/200*1e6:.1f}us")
