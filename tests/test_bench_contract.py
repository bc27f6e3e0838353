"""bench.py's reference arm (the unmodified reference, oracle/_ref, on the host cores):
stdout carries exactly one JSON line with the driver's keys (CPU only)."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(not os.path.exists(os.path.join(ROOT, "oracle", "_ref", "libooc_ref.so")),
                    reason="oracle/_ref not built")
def test_reference_arm_prints_one_json_line():
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"],
                       cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in line, k
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["e2e"]["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_exit_quietly():
    """Under torchrun the reference arm runs on rank 0 only: any other rank exits 0 at once,
    prints nothing and needs no GPU or process group."""
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                        "--warmup", "1"], cwd=ROOT, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    assert r.stdout.strip() == ""


@pytest.mark.gpu
def test_slab_bench_under_torchrun_single_rank():
    """The multi-GPU bench path (torchrun, NCCL, dim-0 slabs, ghost exchange after every
    chain, in core and out of core) on one GPU (OOC_BENCH_FORCE_DIST=1), small grid: one
    JSON line, dp1 slabs."""
    env = dict(os.environ, OOC_BENCH_FORCE_DIST="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", "29541", "bench.py", "--gpus", "1",
           "--size", "2048", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-parity"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["value"] > 0 and line["gpu_launches"] > 0
    assert line["config"]["parallelism"].startswith("dp1 dim-0 slabs")
    # the out-of-core slab path (windowed tiled_explicit runtime on an NCCL communicator)
    assert line["e2e"]["value"] > 0 and "dim-0 slabs" in line["e2e"]["mode"]


@pytest.mark.gpu
def test_bench_two_ranks_on_one_gpu_decompose_one_mesh():
    """bench.py --gpus 2 under torchrun with both ranks on one GPU (gloo for the bench's
    own collectives, the engine's CUDA-IPC transport for the ghost bands): the in-core run
    and the out-of-core e2e run both decompose ONE (2n) x n mesh into dim-0 slabs with
    real neighbour exchanges; one JSON line with dp2 slabs and an e2e value."""
    env = dict(os.environ, OOC_BENCH_BACKEND="gloo", OOC_COMM="ipc")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29543", "bench.py", "--gpus", "2",
           "--size", "1536", "--steps", "2", "--warmup", "3", "--no-cpu", "--no-parity"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = r.stdout.splitlines()
    assert len(lines) == 1, r.stdout
    line = json.loads(lines[0])
    assert line["n_gpus"] == 2 and line["value"] > 0 and line["e2e"]["value"] > 0
    assert line["config"]["parallelism"].startswith("dp2 dim-0 slabs")
    assert "one 3072x1536 mesh in 2 dim-0 slabs" in line["e2e"]["mode"]
