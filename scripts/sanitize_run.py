"""Small end-to-end runs for compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Runs the hot path through the C ABI on C1 (every mode, every regroup engine), a ragged-tile
graph, row lengths straddling the row-pass tile, a long path and star, and an R-MAT 12 graph
(BFS route), and checks labels against the oracle, so a sanitizer report comes with a
functional check of the same launches.

usage (GPU box): compute-sanitizer --tool memcheck python scripts/sanitize_run.py [--quick]
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import graphgen  # noqa: E402
import oracle  # noqa: E402
import paper_1607_06156_b200 as cc  # noqa: E402


def straddle(seed=0):
    rng = np.random.default_rng(77 + seed)
    sizes = [1, 2, 3, 31, 33, 255, 256, 257, 2047, 2048, 2049, 2303, 2305, 4097] * 2
    n = int(sum(sizes) + len(sizes) + 100)
    perm = rng.permutation(n).astype(np.uint32)
    edges, nxt = [], 0
    for s in sizes:
        c = perm[nxt]
        leaves = perm[nxt + 1:nxt + s]
        edges.append(np.stack([np.full(leaves.shape[0], c, np.uint32), leaves], 1))
        nxt += s
    joins = rng.choice(perm[:nxt], size=(len(sizes) // 2, 2)).astype(np.uint32)
    return n, np.concatenate(edges + [joins]).astype(np.uint32)


def main():
    quick = "--quick" in sys.argv
    graphs = [("c1", *(lambda g: (g.n, g.edges))(graphgen.make("c1", 0.25 if quick else 1.0))),
              ("ragged", 3000, graphgen.er(8191, 3000, 8191)),
              ("straddle", *straddle()),
              ("rmat12", *(lambda g: (g.n, g.edges))(graphgen.rmat_scale_graph(12)))]
    n = 20000
    perm = np.random.default_rng(3).permutation(n).astype(np.uint32)
    graphs.append(("path", n, np.stack([perm[:-1], perm[1:]], 1)))
    graphs.append(("star", n, np.stack([np.full(n - 1, 7, np.uint32),
                                        np.delete(np.arange(n, dtype=np.uint32), 7)], 1)))
    engines = ["csr"] if quick else ["csr", "sort", "direct"]
    bad = 0
    for eng in engines:
        ctx = cc.CC(device=0, flags=cc.CC_FLAG_TRACE | cc.REGROUP_FLAGS[eng])
        try:
            for name, nv, e in graphs:
                want = oracle.uf_labels(nv, e)
                ctx.load(e, nv)
                for mode in ("auto", "sv", "bfs+sv"):
                    ctx.run(mode)
                    ok = np.array_equal(ctx.labels(), want)
                    bad += not ok
                    print(f"{eng:7s} {name:9s} {mode:7s} {'ok' if ok else 'MISMATCH'}", flush=True)
        finally:
            ctx.close()
    print("sanitize_run:", "ok" if not bad else f"{bad} mismatches")
    return 1 if bad else 0


if __name__ == "__main__":
    sys.exit(main())
