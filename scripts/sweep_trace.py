"""CTA schedule of the sweep kernels (debug): runs miniflow2d resident with
OOC_SWEEP_TRACE set and summarises, per 14-loop launch of the last chain, the SM idle
fraction, the CTA duration spread and where the idle time sits.

    OOC_GRAPHS=0 OOC_SWEEP_TRACE=gpurun_out/trace.txt python scripts/sweep_trace.py [n]
"""
import os
import sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 15360
path = os.environ["OOC_SWEEP_TRACE"]
if os.path.exists(path):
    os.remove(path)
import paper_1709_02125_b200 as B  # noqa: E402

rt = B.Runtime("resident")
app = sys.argv[2] if len(sys.argv) > 2 else "miniflow2d"
nz = n if app.endswith("3d") else 0
rt.declare_app(app, n, n, nz)
for c in range(3):
    rt.app_iterations(app, n, n, nz, 10 * c, 10 * (c + 1))
    rt.sync()
rt.close()

launches = defaultdict(list)
heads = {}
for line in open(path):
    if line.startswith("#"):
        f = line.split()
        heads[int(f[2])] = line.strip()
        continue
    l, i, sm, t0, t1 = map(int, line.split())
    launches[l].append((i, sm, t0, t1))
last = sorted(launches)[-6:]
for l in last:
    rows = launches[l]
    k0 = min(r[2] for r in rows)
    k1 = max(r[3] for r in rows)
    span = k1 - k0
    per_sm = defaultdict(list)
    for i, sm, t0, t1 in rows:
        per_sm[sm].append((t0 - k0, t1 - k0))
    busy = 0
    first_idle = []
    for sm, iv in per_sm.items():
        iv.sort()
        # union of intervals (2 CTAs per SM overlap)
        cur0, cur1, tot = None, None, 0
        for a, b in iv:
            if cur1 is None or a > cur1:
                if cur1 is not None:
                    tot += cur1 - cur0
                cur0, cur1 = a, b
            else:
                cur1 = max(cur1, b)
        tot += cur1 - cur0
        busy += tot
        first_idle.append(cur1)
    dur = sorted(t1 - t0 for _, _, t0, t1 in rows)
    nsm = len(per_sm)
    print(heads.get(l, l))
    print(f"  span {span/1e3:.1f} us, SMs {nsm}, SM busy (any CTA) {busy / (nsm * span):.3f}, "
          f"CTA us min/median/max {dur[0]/1e3:.1f}/{dur[len(dur)//2]/1e3:.1f}/{dur[-1]/1e3:.1f}, "
          f"SM last-finish min/median {min(first_idle)/1e3:.1f}/{sorted(first_idle)[nsm//2]/1e3:.1f} us")
    # slot occupancy: CTA-slots busy (2 per SM) over the span
    slot_busy = sum(t1 - t0 for _, _, t0, t1 in rows) / (2 * nsm * span)
    starts = sorted(t0 - k0 for _, _, t0, _ in rows)
    print(f"  CTA-slot occupancy {slot_busy:.3f}; first start spread {starts[0]/1e3:.1f}..{starts[min(len(starts), 2*nsm)-1]/1e3:.1f} us")
    conc = defaultdict(int)
    for _, sm, _, _ in rows:
        pass
    # concurrent CTAs per SM (max over time, sampled at CTA starts)
    mx = 0
    for sm, iv in per_sm.items():
        for a, _ in iv:
            mx = max(mx, sum(1 for x, y in iv if x <= a < y))
    print(f"  max concurrent CTAs per SM {mx}")
