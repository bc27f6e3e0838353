"""Out-of-core e2e (miniflow2d 15360^2, capacity = problem/3) with / without prefetch
and cyclic, to measure the streaming engine. One JSON line per configuration."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
import paper_1709_02125_b200 as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
for prefetch in (True, False):
    for cyclic in (True, False):
        r = bench.run_e2e(B, n, 3, 2, 0, cyclic=cyclic, prefetch=prefetch)
        r.pop("clocks", None)
        r["prefetch"], r["cyclic"] = prefetch, cyclic
        r["GBps"] = r["bytes"] / r["wall"] / 1e9
        r["h2d_GBps"] = r["uploaded"] / r["wall"] / 1e9
        print(json.dumps(r), flush=True)
