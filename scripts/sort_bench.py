"""the regroup primitive alone -- the library's onesweep LSD radix sort of
random 64-bit keys with a u32 payload against torch.sort (CUB DeviceRadixSort) on one B200.
PAPER.md:389 benchmarks its samplesort on 2 billion random 64-bit integers.

    python scripts/sort_bench.py [--log2n 30 | --n 2000000000] [--reps 3]

--n 2000000000 is the paper's size; it stays below INT_MAX, which torch.sort needs.
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1607_06156_b200 as cc  # noqa: E402


def timed(fn, reps):
    ts = []
    for _ in range(reps + 1):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    return min(ts[1:])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30,
                    help="torch.sort takes at most INT_MAX elements: 30 for the comparison")
    ap.add_argument("--n", type=int, default=0, help="key count (overrides --log2n)")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    n = args.n or (1 << args.log2n)
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(1607)
    src = torch.randint(-2**63, 2**63 - 1, (n,), dtype=torch.int64, device=dev, generator=g)
    out = {"n": n, "key_bits": 64}
    # ours: keys + u32 payload, 8 passes of 8 bits
    keys, tk = torch.empty_like(src), torch.empty_like(src)
    vals = torch.empty(n, dtype=torch.int32, device=dev)
    tv = torch.empty_like(vals)

    def ours():
        keys.copy_(src)
        vals.copy_(torch.arange(n, dtype=torch.int32, device=dev))
        cc.cc_radix_sort_pairs(keys, vals, tk, tv, 64)
    copy_ms = timed(lambda: (keys.copy_(src), vals.copy_(torch.arange(n, dtype=torch.int32, device=dev))),
                    args.reps)
    ms = timed(ours, args.reps) - copy_ms
    flipped = keys ^ torch.tensor(-2**63, dtype=torch.int64, device=dev)  # unsigned order
    ok = bool(torch.all(flipped[1:] >= flipped[:-1]).item())
    del flipped
    out["onesweep_ms"] = ms
    out["onesweep_Gkeys_s"] = n / ms / 1e6
    out["onesweep_sorted_unsigned"] = ok
    # bytes of an LSD pass: read + write key and payload (histogram pass reads keys once)
    out["onesweep_GBps"] = (n * 8 + 8 * n * 2 * 12) / (ms / 1e3) / 1e9
    del keys, tk, vals, tv
    torch.cuda.empty_cache()
    # CUB through torch.sort (stable; keys + int64 indices)
    ms_t = timed(lambda: torch.sort(src, stable=True), args.reps)
    out["torch_sort_ms"] = ms_t
    out["torch_sort_Gkeys_s"] = n / ms_t / 1e6
    print(json.dumps(out))


if __name__ == "__main__":
    main()
