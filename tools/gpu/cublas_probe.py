import torch
dev = torch.device("cuda:0")
for b, k, h in [(32, 1024, 8192), (32, 2048, 8192)]:
    w = torch.randn((h, k), device=dev).to(torch.bfloat16)
    x = torch.randn((b, k), device=dev).to(torch.bfloat16)
    out = torch.empty((b, h), device=dev, dtype=torch.bfloat16)
    for _ in range(3):
        torch.matmul(x, w.T, out=out)
    torch.cuda.synchronize()
