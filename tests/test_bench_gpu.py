"""bench.py contract on the B200 (our arm): one JSON line with the keys the
driver reads -- metric / value / unit / timing, the roofline object, the
end-to-end (host-buffer) figure with its copy byte counts, clocks, the
launch count and the CPU baseline -- on a reduced grid so the test is fast."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("config,n", [("4", 128), ("5", 96), ("2", 96), ("3", 1024), ("1", 1 << 16)])
def test_bench_line_contract(config, n):
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", config, "--n", str(n),
           "--steps", "4", "--warmup", "3", "--no-ablation", "--no-configs", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config", "e2e",
              "gpu_launches", "roofline", "clocks", "cpu_baseline"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 4 and d["warmup"] == 3
    assert d["value"] > 0 and d["ms_per_step"] > 0 and d["higher_is_better"] is True
    assert d["gpu_launches"] >= 4
    assert "workload" in d["config"]
    rf = d["roofline"]
    assert rf["bound"] == "hbm" and rf["unit"] == "GB/s" and rf["peak"] > 0
    assert abs(rf["frac"] - rf["achieved"] / rf["peak"]) < 1e-9
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    if config in ("5", "2"):  # the host-state sweep, the per-step accumulating ABI beside it
        assert e["mode"] == "sweep" and e["accumulating_abi"]["value"] > 0
        # (--e2e-steps 1: the sweep's one-off copies are not amortised at all)
        assert e["h2d_bytes_per_step"] <= e["accumulating_abi"]["h2d_bytes_per_step"]
    else:
        assert e["mode"] == "abi"
    cb = d["cpu_baseline"]
    assert cb["value"] > 0 and cb["cores"] >= 1 and cb["kind"] in ("reference", "port")
    assert d["clocks"]["samples"] >= 0


def test_bench_fp64_row_and_other_config():
    """The default line also carries the fp64 row (the reference's precision)
    and cfg 4 at the same N."""
    cmd = [sys.executable, os.path.join(ROOT, "bench.py"), "--config", "5", "--n", "96",
           "--steps", "3", "--warmup", "3", "--no-ablation", "--e2e-steps", "1"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([x for x in r.stdout.splitlines() if x.startswith("{")][0])
    assert d["fp64"]["value"] > 0 and d["fp64"]["e2e"]["h2d_bytes_per_step"] > 0
    assert d["cpu_baseline"]["one_thread"]["value"] > 0


@pytest.mark.parametrize("config,halo", [("5", "ipc"), ("4", "ipc"), ("5", "torch")])
def test_bench_two_ranks_one_gpu(config, halo):
    """The N > 1 path end to end -- z-slab plan, pipelined exchange, the
    bitwise check against the exchange-then-compute path, max-over-ranks
    timing, the per-rank e2e with its exchange -- as two ranks on the one GPU
    (gloo for the plumbing; the IPC transport's ordering is stream memory
    operations, no kernel waits on the other rank).  Not a performance run."""
    import socket
    if halo == "torch":
        pytest.skip("torch halo needs NCCL between distinct GPUs")
    so = socket.socket()
    so.bind(("127.0.0.1", 0))
    port = so.getsockname()[1]
    so.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port),
           os.path.join(ROOT, "bench.py"), "--gpus", "2", "--config", config, "--size", "96",
           "--steps", "4", "--warmup", "3", "--halo", halo, "--e2e-steps", "1"]
    env = dict(os.environ, SGB_BENCH_DIST_BACKEND="gloo")
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT, env=env)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["value"] > 0
    assert "bitwise equal" in d["config"]["halo_check"]
    assert "sgb_slab" in d["config"]["halo_exchange"]
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and "z-slab plan" in d["e2e"]["path"]
