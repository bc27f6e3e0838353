import json, time
import paper_1709_02125_b200 as B
from oracle import programs as P
prog = P.app_program("miniflow2d", 64, 64, iters=10)
rt = B.load_program(B.Runtime("plan_only", record=True, tiles=1), prog)
c = rt.num_chains() - 1
t=time.time()
out = rt.chain_sweep_check(c, compile=True)
print(time.time()-t)
for g in out:
    print(g["first"], g["loops"], g["ok"], json.dumps(g["plan"])[:1500] if g["ok"] else g["plan"][:3000])
