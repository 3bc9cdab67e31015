import torch
x = torch.ones(1 << 16, device="cuda")
x.cumsum_(0)
torch.cuda.synchronize()
print("cumsum last", float(x[-1]), "expected", float(1 << 16))
y = torch.ones(1 << 12, 1 << 4, device="cuda")
s = y.sum(0)
y.add_(s)  # in place with a reduction input
print("sum", float(y[0, 0]))
