"""bench.py end to end on the GPU: the single-process contract line, and the multi-process
(torchrun) path in the one-GPU test mode (TIDE_BENCH_SAME_DEVICE: every rank on cuda:0,
gloo process group) for replicas and for peer-memory expert parallelism."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _line(out: str) -> dict:
    lines = [ln for ln in out.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, out[-2000:]
    return json.loads(lines[0])


def test_bench_single_process_contract():
    r = subprocess.run([sys.executable, "bench.py", "--layers", "2", "--steps", "4", "--warmup", "3",
                        "--cpu-seconds", "1"], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
                "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
                "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["value"] > 0 and d["gpu_launches"] > 0 and d["n_gpus"] == 1
    assert d["roofline"]["bound"] == "hbm" and 0 < d["roofline"]["frac"] < 1.2
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] > 0


@pytest.mark.parametrize("extra", [["--replicas"], [], ["--strong"]])
def test_bench_torchrun_two_ranks_one_gpu(extra):
    """torchrun x2 in the one-GPU test mode: replicas, and the N>1 default (flash-shaped
    expert parallelism over peer memory, NVLink accounting) on a 2-layer stack."""
    env = dict(os.environ, TIDE_BENCH_SAME_DEVICE="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--layers", "2", "--steps", "3", "--warmup", "3", "--no-cpu", "--no-e2e"] + extra
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
    ep = "--replicas" not in extra
    assert ("expert parallel x2" in d["config"]["parallelism"]) == ep
    assert d["scaling"] == ("strong" if "--strong" in extra else "weak")
    if "--strong" in extra:  # 8 blocks in total, split over the 2 ranks
        assert d["config"]["tokens_per_layer_step_per_rank"] == 128
    if ep:
        assert "flash" in d["config"]["workload"] and d["nvlink"]["bytes_out_per_layer_step"] > 0
        # the run's own check: EP output over both ranks' tokens == the single-device step
        assert d["ep_check"]["pass"] and d["ep_check"]["bitwise_equal_single_device"], d["ep_check"]
        assert 0 < d["roofline"]["frac"] < 1.2


def test_bench_gpus_flag_spawns_ranks():
    """`python bench.py --gpus 2` (no torchrun) launches the two ranks itself."""
    env = dict(os.environ, TIDE_BENCH_SAME_DEVICE="1")
    env.pop("WORLD_SIZE", None)
    cmd = [sys.executable, "bench.py", "--gpus", "2", "--replicas", "--layers", "2", "--steps", "3",
           "--warmup", "3", "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-2000:]
    d = _line(r.stdout)
    assert d["n_gpus"] == 2 and d["value"] > 0
