"""One K6 launch of a given (batch, k, hidden) for compute-sanitizer runs
(e.g. OFB_K6_SPLITS=8 compute-sanitizer --tool synccheck python tools/k6_sync_case.py 32 1024 2048)."""
import sys, torch
sys.path.insert(0, "/root/repo")
from paper_2601_10729_b200.collective import OprojAllReduce
dev = torch.device("cuda:0")
bsz, k, h = [int(x) for x in sys.argv[1:4]]
w = (torch.randn((2, h, k), device=dev) * k ** -0.5).to(torch.bfloat16)
x = torch.randn((2, bsz, k), device=dev).to(torch.bfloat16)
OprojAllReduce(w, bsz)(x, 1)
torch.cuda.synchronize()
print("ok", bsz, k, h)
