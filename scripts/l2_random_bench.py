"""Reference rates for what bounds the SV row passes: random 4-byte gathers
and random 4-byte atomic-min updates into an n-slot u32 array (C2: n = 16 M, 64 MB, about
half the L2), for L = 49.9 M accesses (one per live tuple of a C2 iteration), timed with
CUDA events using PyTorch's own kernels (index_select, scatter_reduce 'amin') -- the same
kind of library reference as MEASURED_PEAKS.json's copy bandwidth.

    python scripts/l2_random_bench.py [--n 16085771] [--L 49895894]
"""
import argparse
import json

import torch


def timed(fn, reps=5):
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
    ap.add_argument("--n", type=int, default=16085771)
    ap.add_argument("--L", type=int, default=49895894)
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev)
    g.manual_seed(7)
    slots = torch.randint(0, 2**30, (args.n,), dtype=torch.int32, device=dev, generator=g)
    idx = torch.randint(0, args.n, (args.L,), dtype=torch.int64, device=dev, generator=g)
    val = torch.randint(0, 2**30, (args.L,), dtype=torch.int32, device=dev, generator=g)
    out = torch.empty(args.L, dtype=torch.int32, device=dev)
    stream_ms = timed(lambda: out.copy_(val))  # the streaming part alone (read 4L + write 4L)
    gather_ms = timed(lambda: torch.index_select(slots, 0, idx, out=out))
    s2 = slots.clone()
    amin_ms = timed(lambda: s2.scatter_reduce_(0, idx, val, "amin"))
    # the same with the indices sorted (sequential slot order): locality bound vs random
    sidx, _ = torch.sort(idx)
    amin_sorted_ms = timed(lambda: s2.scatter_reduce_(0, sidx, val, "amin"))
    res = {"n": args.n, "L": args.L, "copy_4B_ms": stream_ms, "gather_ms": gather_ms,
           "amin_scatter_ms": amin_ms, "amin_scatter_sorted_ms": amin_sorted_ms,
           "gather_G_per_s": args.L / gather_ms / 1e6, "amin_G_per_s": args.L / amin_ms / 1e6,
           "note": "index_select reads 8-byte indices; scatter_reduce reads 8-byte indices and "
                   "4-byte values per update"}
    print(json.dumps(res))


if __name__ == "__main__":
    main()
