"""bench.py's JSON contract on the GPU, including the N > 1 path.

The N = 2 case runs two torchrun ranks on the box's one GPU with the gloo backend
(bench.py's BF_BENCH_SHARE_GPU / BF_BENCH_DIST_BACKEND test hooks): the ranks never
wait on one another on the device, so this exercises the sharding, W broadcast and
max-over-ranks reduction of the real bench end to end.  Small configs keep it quick.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():   # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
KEYS = ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
        "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
        "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks", "parity")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(args, world=1, timeout=600):
    env = dict(os.environ)
    if world == 1:
        cmd = [sys.executable, "bench.py", *args]
    else:
        env.update(BF_BENCH_SHARE_GPU="1", BF_BENCH_DIST_BACKEND="gloo")
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={world}", "--master-addr", "127.0.0.1",
               "--master-port", str(_port()), "bench.py", "--gpus", str(world), *args]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=timeout)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_c2_single_gpu_contract():
    d = _run(["--config", "c2", "--steps", "5", "--warmup", "3", "--cpu-seconds", "1",
              "--e2e-steps", "2"])
    for k in KEYS:
        assert k in d, k
    assert d["n_gpus"] == 1 and d["unit"] == "REs/s" and d["value"] > 0
    assert d["config"]["workload"] == "c2"
    assert d["roofline"]["bound"] in ("hbm", "alu") and 0 < d["roofline"]["frac"] < 1.5
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["parity"]["ok"] and d["parity"]["blocks"] == 770          # every block vs the oracle
    srv = d["server"]
    assert srv["bitwise_equal_to_bf_apply"] and 0 < srv["device_us_median"] < 1000
    assert d["e2e"]["h2d_bytes_per_step"] == 770 * 480 * 36
    assert d["e2e"]["d2h_bytes_per_step"] == 770 * 30720
    assert d["gpu_launches"] >= 5
    assert d["config"]["submission"] == "cuda_graph"
    assert "split precision" in d["config"]["arith"]


def test_bench_filter_contract():
    d = _run(["--config", "fl1", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1",
              "--e2e-steps", "1"])
    for k in KEYS:
        assert k in d, k
    assert d["unit"] == "samples/s" and d["value"] > 0
    assert 0 < d["roofline"]["frac"] < 1.2 and d["roofline"]["traffic"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == d["e2e"]["d2h_bytes_per_step"] == (1 << 18) * 2048 * 8


def test_bench_c4_two_ranks_share_gpu():
    """torchrun N = 2: subband sharding, W broadcast, max over ranks, whole-job value."""
    d = _run(["--config", "c4", "--steps", "3", "--warmup", "3", "--no-e2e", "--steady-seconds", "0",
              "--parity-stride", "256"], world=2)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2")
    assert d["config"]["world_size"] == 2 and d["config"]["backend"] == "gloo"
    assert d["cpu_baseline"] is None          # rank 0 at N = 1 only
    assert d["gpu_launches"] >= 2 * 3
    par = d["parity"]                         # every rank checked its own shard
    assert par["ok"] and len(par["per_rank"]) == 2 and all(r["ok"] and r["blocks"] > 0 for r in par["per_rank"])


def test_bench_c5_short_stream():
    d = _run(["--config", "c5", "--steps", "3", "--warmup", "3", "--c5-chunks", "64"])
    assert d["config"]["workload"] == "c5" and d["config"]["chunks_per_step"] == 64
    assert d["config"]["launch_mode"] == "cuda_graph"
    assert d["config"]["chunks_per_launch"] == 16 and d["config"]["launches_per_step"] == 4
    assert d["config"]["apply_sms"] + d["config"]["route_sms"] \
        == torch.cuda.get_device_properties(0).multi_processor_count
    assert d["value"] > 0 and 0 < d["roofline"]["frac"] < 1.5


def test_bench_c5_two_ranks_windows():
    """torchrun N = 2 on c5: whole 16-chunk windows dealt to the ranks, every rank's ring
    checked against the oracle."""
    d = _run(["--config", "c5", "--steps", "2", "--warmup", "3", "--c5-chunks", "64"], world=2)
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["parallelism"].startswith("dp2 (whole 16-chunk windows")
    assert d["config"]["launches_per_step"] == 2            # this rank's windows: 4 / 2
    par = d["parity"]
    assert par["ok"] and len(par["per_rank"]) == 2 and all(r["blocks"] > 0 for r in par["per_rank"])


def test_bench_ofdm_contract():
    d = _run(["--config", "of0", "--steps", "3", "--warmup", "3", "--cpu-seconds", "1",
              "--e2e-steps", "1"])
    for k in KEYS:
        assert k in d, k
    assert d["unit"] == "REs/s" and d["value"] > 0 and d["config"]["workload"] == "of0"
    assert d["parity"]["ok"] and d["parity"]["blocks"] == 6 * 64      # every symbol, all antennas
    assert d["roofline"]["kernel"] in d["roofline"]["kernels"]
    assert d["e2e"]["d2h_bytes_per_step"] == 6 * 64 * (144 + 2048) * 8
    assert d["gpu_launches"] >= 2 * 3


def test_bench_ofdm_two_ranks_share_gpu():
    d = _run(["--config", "of0", "--steps", "2", "--warmup", "3", "--no-e2e"], world=2)
    assert d["n_gpus"] == 2 and d["value"] > 0 and d["cpu_baseline"] is None
    par = d["parity"]
    assert par["ok"] and len(par["per_rank"]) == 2 and all(r["blocks"] == 3 * 64 for r in par["per_rank"])


def test_bench_ofdm_reference_arm():
    d = _run(["--impl", "reference", "--config", "of0", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["config"]["workload"] == "of0"


def test_bench_reference_arm():
    d = _run(["--impl", "reference", "--config", "c2", "--steps", "2", "--warmup", "3",
              "--cpu-seconds", "1"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0
