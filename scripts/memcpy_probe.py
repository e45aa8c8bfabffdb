import torch, time
h = torch.empty(1024, dtype=torch.uint8).pin_memory()
d = torch.empty(1024, dtype=torch.uint8, device='cuda')
x = torch.empty(1 << 20, device='cuda')
s = torch.cuda.Stream()
with torch.cuda.stream(s):
    for rep in range(3):
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for i in range(100):
            d.copy_(h, non_blocking=True)
        e1.record(); e1.synchronize()
        print("100 H2D 1KB copies: %.2f us each" % (e0.elapsed_time(e1) * 10))
        e0.record()
        for i in range(100):
            x.add_(1.0)
        e1.record(); e1.synchronize()
        print("100 tiny kernels: %.2f us each" % (e0.elapsed_time(e1) * 10))
        e0.record()
        for i in range(100):
            d.copy_(h, non_blocking=True); x.add_(1.0)
        e1.record(); e1.synchronize()
        print("100 copy+kernel pairs: %.2f us each" % (e0.elapsed_time(e1) * 10))
