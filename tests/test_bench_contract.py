"""bench.py's JSON contract: the reference arm runs anywhere (CPU oracle
port); the GPU arm's line carries every key the driver reads."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def run(args, timeout=600):
    p = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], cwd=ROOT,
                       capture_output=True, text=True, timeout=timeout)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, p.stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = run(["--impl", "reference", "--steps", "2", "--warmup", "1"])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["steps"] == 2 and d["warmup"] == 1 and d["higher_is_better"] is True
    assert d["cpu_baseline"]["kind"] in ("port", "reference") and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"] == {"value": d["value"], "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]


@pytest.mark.gpu
def test_gpu_arm_line():
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = run(["--steps", "300", "--warmup", "3", "--no-cpu-baseline", "--ttft-layers", "4"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "roofline", "e2e", "gpu_launches", "clocks"):
        assert k in d, k
    assert d["steps"] == 300 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and 0 < r["frac"] < 1.2
    assert abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert e["bit_exact_vs_device_call"] is True
    assert d["gpu_launches"] >= d["steps"]
    assert "workload" in d["config"] and "model" not in d["config"]
    g = d["producer_gemm"]
    for shp in ("o_proj_tp2", "down_proj_tp2"):
        assert g[shp]["shard_equals_k1_of_own_partial"] is True
        # a GEMM of >= 17 GFLOP cannot take under 5 us: guards against a
        # timed graph that captured nothing
        assert g[shp]["fused_gemm_quant_us"] > 5 and g[shp]["cublas_plus_k1_us"] > 5
    t1 = d["ttft"]["tp1"]
    assert t1["layers"] == 4 and t1["bf16"]["ms"] > 0 and t1["mx_fused_gemm"]["ms"] > 0
    assert "codec_overhead_pct" in t1["mx_unfused"] and "codec_overhead_pct" in t1["mx"]


@pytest.mark.gpu
def test_gpu_arm_world1_nccl_line():
    """--force-dist: a world-1 NCCL process group runs the TP=N code path end
    to end (NCCL collectives, the NVLink kernels over real symmetric memory,
    the TTFT block with every all-reduce variant)."""
    torch = pytest.importorskip("torch")
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    d = run(["--steps", "60", "--warmup", "3", "--force-dist", "--ttft-layers", "2",
             "--no-70b"])
    assert d["n_gpus"] == 1 and d["value"] > 0
    assert d["collective"] is not None
    lc = d["linear_collective"]
    assert lc["mx_push_bit_exact_vs_mx_nccl"] is True, lc
    assert lc["bf16_nccl_us"] > 0 and lc["mx_nccl_us"] > 0 and lc["mx_push_us"] > 0
    t = d["ttft"]["llama-3.1-8b"]
    assert t["layers"] == 2
    for k in ("bf16_nccl", "mx_oneshot", "mx_oneshot_unfused", "mx_twoshot", "mx_symm", "mx_symm2",
              "mx_push", "mx_paper_scheme", "mx_paper_scheme_push"):
        assert "ms" in t[k], (k, t[k])


def test_deadline_prints_partial_line_and_exits_zero():
    """The watchdog: once the headline line exists, an overrunning block
    ends the run with that line (plus ``truncated``) and exit status 0; a
    run that finishes in time prints the line exactly once."""
    code = ("import sys, time; sys.path.insert(0, %r); import bench; "
            "d = bench.Deadline(time.time(), %s, 0); d.at('ttft'); "
            "d.line = {'metric': 'm', 'value': 1.0}; %s")
    p = subprocess.run([sys.executable, "-c", code % (ROOT, 1.0, "time.sleep(30)")],
                       capture_output=True, text=True, timeout=60)
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] == 1.0 and "'ttft'" in d["truncated"]
    p = subprocess.run([sys.executable, "-c",
                        code % (ROOT, 30.0, "d.put(ttft=None); d.emit(); d.emit()")],
                       capture_output=True, text=True, timeout=60)
    assert p.returncode == 0
    lines = [l for l in p.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1 and "truncated" not in json.loads(lines[0])
