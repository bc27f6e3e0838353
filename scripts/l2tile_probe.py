"""Host vs device time of the L2-tiled in-core mode (config 2 tiled)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_02125_b200 as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
budget = int(sys.argv[2]) if len(sys.argv) > 2 else 96 << 20
rt = B.Runtime("resident", resident_budget=budget)
rt.declare_app("miniflow2d", n, n)
rt.app_iterations("miniflow2d", n, n, 0, 0, 60)  # 6 chains: tuning + graph capture
rt.sync()
d0 = rt.device(); r0 = rt.report()
m0 = rt.mark(); t0 = time.perf_counter()
rt.app_iterations("miniflow2d", n, n, 0, 60, 70)
t_issue = time.perf_counter() - t0
m1 = rt.mark(); rt.sync(); wall = time.perf_counter() - t0
d1 = rt.device(); r1 = rt.report()
print(json.dumps({"budget": budget, "tiles": r1["tiles"], "device_s": rt.elapsed(m0, m1), "wall_s": wall,
                  "issue_s": t_issue, "launches": d1["kernel_launches"] - d0["kernel_launches"],
                  "jit_host_s": (d1["jit_host_us"] - d0["jit_host_us"]) * 1e-6,
                  "graph_launches": d1["graph_launches"] - d0["graph_launches"],
                  "GBps": (r1["total_bytes"] - r0["total_bytes"]) / rt.elapsed(m0, m1) / 1e9}))
