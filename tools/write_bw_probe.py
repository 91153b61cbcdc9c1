import torch
n = 6 * 805306368
a = torch.empty(n, dtype=torch.int32, device='cuda')
b = torch.empty(805306368, dtype=torch.int32, device='cuda')
for _ in range(3): a.fill_(1)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5): a.fill_(7)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print('fill 19.3 GB: %.2f ms = %.2f TB/s' % (ms, n * 4 / ms / 1e9))
# read 3.2 GB + write 19.3 GB: broadcast copy
v = a.view(6, -1)
e0.record()
for _ in range(5): v.copy_(b.view(1, -1).expand(6, -1))
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print('read 3.2 + write 19.3 GB (broadcast copy): %.2f ms = %.2f TB/s' % (ms, (n * 4 + 805306368 * 4) / ms / 1e9))
