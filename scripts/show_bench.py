"""Print the essentials of bench.py JSON lines: python scripts/show_bench.py <file>..."""
import json
import sys

for f in sys.argv[1:]:
    for ln in open(f):
        ln = ln.strip()
        if not ln.startswith("{"):
            continue
        d = json.loads(ln)
        c = d.get("config", {})
        print(f, c.get("workload", "")[:24], c.get("mode"), c.get("regroup"), "route", c.get("route"),
              "iters", c.get("sv_iterations"))
        print(f"  value {d['value'] / 1e9:.3f} G/s  ms/step {d['ms_per_step']:.3f}  launches {d.get('gpu_launches')}")
        r = d.get("roofline") or {}
        print(f"  roofline {r.get('kernel')}: {r.get('achieved', 0) or 0:.0f} GB/s frac {r.get('frac')} "
              f"share {r.get('share_of_step')} ms/launch {r.get('ms_per_launch')}")
        if d.get("path_roofline"):
            print(f"  path frac {d['path_roofline']['frac']:.3f}  stages {d.get('stages_ms')}")
        if d.get("e2e"):
            print(f"  e2e {d['e2e']['value'] / 1e9:.3f} G/s match {d.get('e2e_labels_match_oracle')} clocks {d.get('clocks')}")
        for k, v in (d.get("kernels") or {}).items():
            print(f"    {k[:48]:48s} {v['ms_per_step']:.3f} ms  {v['alg_GBps'] or 0:.0f} GB/s  x{v['launches_per_step']}")
