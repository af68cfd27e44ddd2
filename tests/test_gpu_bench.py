"""bench.py's contract, run as the driver runs it: one JSON line on rank 0 with
the keys the round-end checks read, for one GPU and (functionally) for two
ranks.  Two ranks share the one GPU of the test box through the gloo backend
(SKV_BENCH_BACKEND / SKV_BENCH_DEVICE): the ranks never wait on each other's
kernels, so this exercises the multi-rank code path (barriers, max over
ranks, the result gather, the head-sharded all-reduce) -- its numbers are not
measurements."""

import json
import os
import socket
import subprocess
import sys

import pytest

torch = pytest.importorskip("torch")

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _cuda():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _json_lines(out: str):
    return [json.loads(x) for x in out.splitlines() if x.startswith("{")]


def _run(cmd, env=None, timeout=600):
    e = dict(os.environ)
    e.update(env or {})
    p = subprocess.run(cmd, cwd=ROOT, env=e, stdout=subprocess.PIPE, stderr=subprocess.PIPE, text=True,
                       timeout=timeout)
    assert p.returncode == 0, p.stderr[-3000:]
    return _json_lines(p.stdout)


def _check_line(d, n):
    for key in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
                "vs_baseline", "dtype", "config", "roofline", "e2e", "gpu_launches", "clocks"):
        assert key in d, key
    assert d["n_gpus"] == n and d["value"] > 0 and d["ms_per_step"] > 0 and d["gpu_launches"] > 0
    assert "workload" in d["config"]
    r = d["roofline"]
    assert r["bound"] in ("hbm", "tensor") and r["achieved"] > 0 and r["peak"] > 0
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0


def test_bench_one_gpu_json_line():
    lines = _run([sys.executable, "bench.py", "--workload", "cfg0", "--steps", "3", "--warmup", "3",
                  "--no-cpu-baseline"])
    assert len(lines) == 1
    _check_line(lines[0], 1)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("workload,extra", [("cfg0", []), ("cfg3", ["--select", "layer"]),
                                            ("cfg3", ["--select", "kv_head"])])
def test_bench_two_ranks_functional(workload, extra):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2", "--master-addr",
           "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2", "--workload", workload,
           "--steps", "3", "--warmup", "3", *extra]
    lines = _run(cmd, env={"SKV_BENCH_BACKEND": "gloo", "SKV_BENCH_DEVICE": "0"}, timeout=900)
    assert len(lines) == 1, "rank 0 alone prints the line"
    d = lines[0]
    _check_line(d, 2)
    if workload == "cfg3":
        assert "sharded x2" in d["config"]["parallelism"]
