"""Write the full-size SV traces of configs C1-C3 (tests/golden/trace_<cfg>.json).

Calls only oracle/ (the Alg. 1 numpy transcription) and graphgen/ (inputs): the stored
values come from the oracle, never from the CUDA path.  Run: python tests/golden/make_traces.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import graphgen  # noqa: E402
from oracle import sv  # noqa: E402


def main(cfgs):
    for cfg in cfgs:
        g = graphgen.make(cfg)
        t = time.time()
        _, tr = sv.sv_trace(g.n, g.edges)
        out = {"config": cfg, "n": g.n, "m": g.m, "generator": "graphgen.make(%r, 1.0)" % cfg,
               "source": "oracle.sv.sv_trace (Alg. 1, PAPER.md:133-178, early exclusion R4)",
               "seconds": round(time.time() - t, 1),
               "trace": [{k: int(v) for k, v in r.items()} for r in tr]}
        with open(os.path.join(ROOT, "tests", "golden", f"trace_{cfg}.json"), "w") as f:
            json.dump(out, f, indent=1)
        print(cfg, len(tr), "iterations", out["seconds"], "s", flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c1", "c2", "c3"])
