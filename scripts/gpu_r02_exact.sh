#!/bin/bash
# Exact-reduction mode: GPU parity tests + timing of the exact fold at the benched size.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_large.py -x -q -m gpu \
  > gpurun_out/r02x_pytest.log 2>&1; echo "rc=$?" >> gpurun_out/r02x_pytest.log
timeout 600 python - > gpurun_out/r02x_time.log 2>&1 <<'PY'
import time
import paper_1709_02125_b200 as B
n = 15360
for exact in (False, True):
    rt = B.Runtime("resident", exact_reductions=exact)
    rt.declare_app("miniflow2d", n, n)
    for c in range(3):
        t0 = time.perf_counter()
        rt.app_iterations("miniflow2d", n, n, 0, 10 * c, 10 * (c + 1))
        v = rt.fetch_reduction("fieldsum")
        print(f"exact={exact} chain {c}: {time.perf_counter() - t0:.3f} s fieldsum {v.hex()}", flush=True)
    print(rt.device())
    rt.close()
PY
echo "rc=$?" >> gpurun_out/r02x_time.log
