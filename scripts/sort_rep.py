"""Repeated in-process timings of cc_radix_sort_pairs (variance study).
usage: python scripts/sort_rep.py [log2n] [reps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_06156_b200 as cc  # noqa: E402

n = 1 << int(sys.argv[1] if len(sys.argv) > 1 else 26)
reps = int(sys.argv[2] if len(sys.argv) > 2 else 8)
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev)
g.manual_seed(int(os.environ.get("SEED", "1607")))
src = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=dev, generator=g)
keys, tk = torch.empty_like(src), torch.empty_like(src)
vals = torch.empty(n, dtype=torch.int32, device=dev)
tv = torch.empty_like(vals)
ts = []
for _ in range(reps):
    keys.copy_(src)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    cc.cc_radix_sort_pairs(keys, vals, tk, tv, 64)
    b.record()
    torch.cuda.synchronize()
    ts.append(round(a.elapsed_time(b), 2))
print(os.environ.get("CC_RADIX_ITEMS", "16"), ts)
