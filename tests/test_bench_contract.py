"""bench.py's JSON contract: the reference arm on CPU (-m "not gpu") and the
GPU arm on a small config (-m gpu), each checked for the keys and units the
driver reads."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(args, timeout=600):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py")] + args,
                         capture_output=True, text=True, timeout=timeout, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_reference_arm_json():
    """--impl reference: the CPU oracle on the same workload config, metric
    and unit as the GPU arm, with the cpu_baseline and e2e blocks."""
    d = _run(["--impl", "reference", "--config", "C1", "--steps", "1", "--warmup", "3"])
    assert d["impl"] == "reference" and d["unit"] == "iterations/s"
    assert d["higher_is_better"] is True and d["value"] > 0
    assert d["config"]["workload"].startswith("C1: 2-D central conv-diff 32^2")
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


@pytest.mark.gpu
def test_gpu_arm_json():
    """The GPU arm on C1: value, roofline (dominant kernel, measured peak,
    fraction), e2e with copied bytes, clocks, launches, CPU baseline."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    d = _run(["--config", "C1", "--steps", "1", "--warmup", "3", "--cpu-sample-iters", "8"])
    assert d["unit"] == "iterations/s" and d["value"] > 0 and d["n_gpus"] == 1
    assert d["steps"] == 1 and d["warmup"] == 3 and d["dtype"] == "f64"
    r = d["roofline"]
    assert r["bound"] == "hbm" and r["unit"] == "GB/s" and r["peak"] > 1000
    assert 0 < r["frac"] == pytest.approx(r["achieved"] / r["peak"])
    assert r["kernel"] in ("fused", "pass1", "pass2")
    e = d["e2e"]
    assert e["value"] > 0 and e["h2d_bytes_per_step"] > 0 and e["d2h_bytes_per_step"] > 0
    assert d["gpu_launches"] > 0
    assert "sm_mhz" in d["clocks"] and isinstance(d["clocks"]["reasons"], list)
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["value"] > 0


def test_algorithmic_byte_formulas():
    """The roofline's algorithmic bytes on C2's sizes, by hand:
    SELL-equivalent matrix pair = 2 (nnz (8 + 4) + 4 (n + 1)), one shared
    column array saves 4 nnz, int16 deltas 2 nnz more; the fused kernel moves
    12 n-vectors, pass 1 / pass 2 (k = 0, lazy x) 8 and 6."""
    sys.path.insert(0, ROOT)
    import bench
    n, nnz = 1048576, 5238784
    mat = 2 * (nnz * 12 + 4 * (n + 1))
    assert bench.alg_bytes_fused(n, nnz, 8, False, False) == mat + 12 * n * 8
    assert bench.alg_bytes_fused(n, nnz, 8, True, False) == mat - 4 * nnz + 12 * n * 8
    assert bench.alg_bytes_fused(n, nnz, 8, True, True) == 203350024
    p1, p2 = bench.alg_bytes(n, nnz, 0, 8, True, True)
    assert p1 == mat - 4 * nnz + 8 * n * 8 and p2 == 6 * n * 8
    p1k, p2k = bench.alg_bytes(n, nnz, 10, 8, True, True)
    assert p1k - p1 == 2 * 10 * n * 8 and p2k - p2 == 2 * 10 * n * 8
