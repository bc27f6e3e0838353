"""Small, deterministic driver for ncu captures: miniflow2d resident (one warm-up
chain + one measured chain of 10 iterations)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1709_02125_b200 as B
n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
fuse = int(sys.argv[2]) if len(sys.argv) > 2 else 1
rt = B.Runtime("resident", fuse=bool(fuse))
rt.declare_app("miniflow2d", n, n)
rt.app_iterations("miniflow2d", n, n, 0, 0, 20)
rt.sync()
print(rt.device())
