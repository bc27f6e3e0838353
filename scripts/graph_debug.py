import sys, os
sys.path.insert(0, os.getcwd())
import paper_1709_02125_b200 as B
B.set_jit(2, 0)
rt = B.Runtime("resident")
rt.run_app("miniflow2d", 200, 180, 0, 52)
print(rt.device())
