"""bench.py's reference arm on the host (no GPU): the JSON line the driver parses.

The reference arm times the CPU oracle (this tier has no reference implementation)
on the same workload, metric and unit as the GPU arm; under torchrun only rank 0 prints.
"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
KEYS = {"impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
        "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"}


def _run(extra_env=None, *args):
    env = dict(os.environ, **(extra_env or {}))
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference", *args],
                          capture_output=True, text=True, env=env, cwd=str(ROOT), timeout=600)


def test_reference_arm_json_line():
    p = _run(None, "--config", "tiny", "--queries", "100", "--steps", "1", "--warmup", "0", "--ref-sample", "20")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert KEYS <= set(d), KEYS - set(d)
    assert d["impl"] == "reference" and d["unit"] == "queries/s" and d["value"] > 0
    assert d["higher_is_better"] is True and d["vs_baseline"] is None
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["config"]["workload"].startswith("tiny") or "tiny" in d["config"]["workload"]


def test_reference_arm_other_ranks_are_silent():
    p = _run({"RANK": "1", "WORLD_SIZE": "2"}, "--config", "tiny", "--steps", "1", "--warmup", "0")
    assert p.returncode == 0, p.stderr[-2000:]
    assert not [ln for ln in p.stdout.splitlines() if ln.startswith("{")]


def test_plumbing_check_two_ranks_gloo():
    """bench.py's N > 1 step plumbing (process group, the all-gather inside each timed step, the
    max over ranks, rank-0 printing) under torchrun with 2 ranks on gloo, a host stand-in for the
    library call.  The gathered results must equal every rank's stand-in values in global order."""
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    p = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
                        "--master-addr", "127.0.0.1", "--master-port", str(port), str(ROOT / "bench.py"),
                        "--plumbing-check", "--gpus", "2", "--queries", "1001", "--steps", "3", "--warmup", "1"],
                       capture_output=True, text=True, cwd=str(ROOT), timeout=600)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, p.stdout
    d = json.loads(lines[0])
    assert d["plumbing_check"] is True and d["n_ranks"] == 2 and d["gathered_ok"] is True


import pytest  # noqa: E402


@pytest.mark.gpu
def test_bench_gpu_line_tiny():
    """The GPU arm end to end on the tiny config: one JSON line with the contract's keys, the
    roofline and cpu_baseline objects, e2e with the bytes copied, launches counted, a sampled
    parity summary with no differences beyond 1e-9."""
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "tiny", "--steps", "3", "--warmup", "3",
                        "--no-spmm"], capture_output=True, text=True, cwd=str(ROOT), timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    need = {"metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
            "vs_baseline", "dtype", "data", "config", "roofline", "cpu_baseline", "e2e", "gpu_launches", "clocks"}
    assert need <= set(d), need - set(d)
    assert d["value"] > 0 and d["e2e"]["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 100 * 8 and d["e2e"]["d2h_bytes_per_step"] == 100 * 8
    for k in ("bound", "achieved", "peak", "unit", "frac"):
        assert k in d["roofline"], k
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    ps = d["parity_summary"]
    assert ps["max_abs_diff_r"] <= 1e-9 and ps["ties"] == 0 and ps["walk_checksums_equal"] == ps["queries"]


@pytest.mark.gpu
def test_bench_gpu_line_tiny_strong_scaling():
    """`--scaling strong` at N = 1: the global query list goes through dist.partition, query_ids and
    the partition-order results; the line names the global list (no per-GPU count) and its sampled
    parity against the oracle is clean."""
    p = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--config", "tiny", "--steps", "3", "--warmup", "3",
                        "--no-spmm", "--scaling", "strong"], capture_output=True, text=True, cwd=str(ROOT),
                       timeout=900)
    assert p.returncode == 0, p.stderr[-3000:]
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["scaling"] == "strong" and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["queries_total"] == 100 and d["config"]["queries_per_gpu"] is None
    assert "queries in all" in d["config"]["workload"]
    ps = d.get("parity_summary")
    if ps:
        assert ps["max_abs_diff_r"] <= 1e-9 and ps["walk_checksums_equal"] == ps["queries"]
