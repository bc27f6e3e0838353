"""Run each miniflow2d loop of iteration 0 alone (own process) through the forced
TMA template; report which ones fail."""
import json, os, subprocess, sys
sys.path.insert(0, os.getcwd())
if len(sys.argv) > 1 and sys.argv[1] != 'all':
    import paper_1709_02125_b200 as B
    from oracle import programs as P
    from tests.helpers import compare, oracle_record, product_record
    B.set_jit(2, 0)
    ks = [int(x) for x in sys.argv[1].split(",")]; n = int(sys.argv[2]) if len(sys.argv) > 2 else 300
    full = P.app_program("miniflow2d", n, 256, 0, iters=1)
    loops = [o for o in full["ops"] if o["op"] == "loop"]
    prog = dict(full); prog["ops"] = [loops[k] for k in ks] + [{"op": "finish"}]
    k = ks
    want = oracle_record(prog, "explicit", tiles=1); want.pop("_rt", None)
    got = product_record(prog, "explicit", tiles=1); got.pop("_rt", None)
    print("loop", k, "diff", str(compare(want, got))[:200], flush=True)
else:
    for k in ["0,0", "0,1", "1,0", "3,3", "0,1,2", "0,1,2,3,4,5", "0,1,2,3,4,5,6,7,8,9,10,11,12,13"]:
        r = subprocess.run([sys.executable, __file__, k], capture_output=True, text=True, timeout=60)
        print(k, r.returncode, (r.stdout + r.stderr).strip().splitlines()[-1][:200], flush=True)
