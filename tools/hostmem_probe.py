"""Does the host-side page size change the H2D link rate?  Best-of-10 1 GiB
cudaMemcpyAsync H2D / D2H from (a) cudaHostAlloc memory (what the arena uses)
and (b) 2 MiB-aligned memory advised as transparent huge pages, pinned with
cudaHostRegister.  Also reports the THP setting of the box."""
import ctypes
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2601_10729_b200 import _native  # noqa: E402
from paper_2601_10729_b200.runtime import link_probe  # noqa: E402

NB = 1 << 30
libc = ctypes.CDLL("libc.so.6", use_errno=True)
lib = _native.load()
dev = torch.device("cuda:0")
d = torch.empty(NB, dtype=torch.uint8, device=dev)
res = {}
try:
    res["thp"] = Path("/sys/kernel/mm/transparent_hugepage/enabled").read_text().strip()
except OSError:
    res["thp"] = None

h = lib.ofb_host_alloc(NB)
res["cudaHostAlloc"] = link_probe(h, d.data_ptr(), NB, 10)
lib.ofb_host_free(h)

p = ctypes.c_void_p()
assert libc.posix_memalign(ctypes.byref(p), 1 << 21, NB) == 0
MADV_HUGEPAGE = 14
res["madvise_rc"] = libc.madvise(p, ctypes.c_size_t(NB), MADV_HUGEPAGE)
ctypes.memset(p, 1, NB)          # fault the pages in (huge where THP allows)
cudart = torch.cuda.cudart()
rc = cudart.cudaHostRegister(p.value, NB, 0)
res["register_rc"] = int(rc) if not isinstance(rc, tuple) else int(rc[0])
try:
    smaps = Path("/proc/self/smaps_rollup").read_text()
    res["AnonHugePages"] = [l for l in smaps.splitlines() if "AnonHugePages" in l]
except OSError:
    pass
res["thp_registered"] = link_probe(p.value, d.data_ptr(), NB, 10)
cudart.cudaHostUnregister(p.value)
print(json.dumps(res))
