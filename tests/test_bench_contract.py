"""bench.py's driver contract on CPU: `--impl reference` (the oracle arm, no GPU) prints ONE
JSON line with the required keys and sane values, and the pure helpers bench.py computes
its roofline from agree with the planner (algorithmic HBM bytes of the loopback schedule)."""
import json
import os
import subprocess
import sys

import pytest

import bench
from paper_1811_12174_b200 import ddl

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REQUIRED = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
            "scaling", "vs_baseline", "dtype", "data", "config")


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, lines
    d = json.loads(lines[0])
    for k in REQUIRED:
        assert k in d, k
    assert d["impl"] == "reference"
    assert d["metric"] == json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    assert d["steps"] == 1 and d["warmup"] == 3 and d["n_gpus"] == 1
    assert d["value"] > 0 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert "workload" in d["config"]


def test_reference_arm_other_ranks_exit_quietly():
    env = dict(os.environ, RANK="1", WORLD_SIZE="2", LOCAL_RANK="1")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--gpus", "2",
                        "--steps", "1", "--warmup", "3"], capture_output=True, text=True, timeout=300, cwd=ROOT,
                       env=env)
    assert r.returncode == 0 and r.stdout.strip() == ""


def test_loopback_algorithmic_bytes_match_planner_traffic():
    """bench.loopback_hbm_bytes (roofline numerator) = per rank: own reads + writes of every
    phase, which for the RS reads is (peer bytes from ddl_plan_traffic) + own block bytes;
    checked against an independent count from the planner's block sets."""
    P, w = 8, 4
    for dims in ([4, 2], [8], [2, 2, 2], [2, 4]):
        for n in (1 << 20, 1_000_003, 2049000):
            got = bench.loopback_hbm_bytes(n, P, dims, w)
            q = ddl.block_elems(n, P, "float32")

            def blen(b):
                return max(0, min(n, (b + 1) * q) - min(n, b * q)) * w
            want = 0
            for r in range(P):
                for d in range(len(dims)):
                    if dims[d] == 1:
                        continue
                    act = ddl.plan_blocks(P, dims, r, d + 1)   # blocks r reduces in RS d / receives in AG d
                    byts = sum(blen(b) for b in act)
                    want += dims[d] * byts + byts              # RS d: read g copies, write one
                    for m in ddl.plan_group(P, dims, r, d):    # AG d: read + write every peer's set
                        if m != r:
                            mb = sum(blen(b) for b in ddl.plan_blocks(P, dims, m, d + 1))
                            want += 2 * mb
            assert got == want, (dims, n, got, want)


N_GT_1_KEYS = ("roofline", "cpu_baseline", "e2e", "nccl", "per_bucket", "clocks", "gpu_launches",
               "correctness_gate")


@pytest.mark.gpu
def test_multi_rank_line_same_gpu():
    """The N > 1 leg (torchrun, one process per rank) produces a complete line: roofline
    (900 GB/s peak + a peer-copy peak measured in the run), cpu_baseline, e2e, nccl (null on
    one GPU: NCCL refuses two ranks per device), per-bucket bus bandwidth.  Run with every
    rank on cuda:0 (DDL_BENCH_SAME_GPU=1) -- a functional check; the numbers mean nothing."""
    env = dict(os.environ, DDL_BENCH_SAME_GPU="1", DDL_TIMEOUT_MS="60000")
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                        "--master-addr", "127.0.0.1", "--master-port", "29631", os.path.join(ROOT, "bench.py"),
                        "--gpus", "2", "--steps", "3", "--warmup", "3"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.strip().startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    for k in REQUIRED + N_GT_1_KEYS:
        assert k in d, k
    assert d["n_gpus"] == 2 and d["config"]["same_gpu"] is True
    assert d["roofline"]["peak"] == 900.0 and d["roofline"]["measured_peer_copy"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0
    assert d["nccl"] is None
    assert len(d["per_bucket"]) == 5 and all(b["busbw"] > 0 for b in d["per_bucket"])
    assert d["e2e"]["h2d_bytes_per_step"] > 0
