"""bench.py's output contract on the GPU (the one JSON line the driver parses): metric / unit / config of
BASELINE.json, the device-timed value consistent with ms_per_step, the end-to-end number through host buffers with
its copy sizes, the kernel-launch count of the timed region, the §8(d) roofline object of the dominant kernel, and
the clocks sampled during the timed region. Runs the default (C3) workload briefly in a subprocess."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.gpu
def test_bench_json_line_contract():
    steps = 3
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--steps", str(steps), "--warmup", "3",
                        "--no-cpu-baseline"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [x for x in r.stdout.splitlines() if x.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = json.loads(lines[0])
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))
    assert d["metric"] == base["metric"]
    assert d["unit"] == "env-steps/s" and d["higher_is_better"] is True and d["scaling"] == "weak"
    assert d["n_gpus"] == 1 and d["steps"] == steps and d["warmup"] >= 3
    assert d["vs_baseline"] is None
    cfg = d["config"]
    assert cfg["n_envs_per_gpu"] == 4096 and cfg["n_steps"] == 24 and cfg["global_batch"] == 98304
    assert "workload" in cfg and "l2" in cfg
    # the device-timed value is the whole job's samples over the max-over-ranks iteration time
    assert d["value"] > 0 and d["ms_per_step"] > 0
    assert abs(d["value"] - 4096 * 24 / (d["ms_per_step"] * 1e-3)) <= 1e-6 * d["value"]
    e2e = d["e2e"]
    assert e2e["unit"] == d["unit"] and e2e["value"] > 0
    assert e2e["h2d_bytes_per_step"] > 0 and e2e["d2h_bytes_per_step"] > 0
    assert e2e["value"] <= 1.1 * d["value"]  # host buffers and a sync every iteration cannot beat the device time
    # the launch count of the timed region: whole iterations of the captured graph
    assert d["gpu_launches"] > 0 and d["gpu_launches"] % steps == 0
    roof = d["roofline"]
    assert roof["bound"] == "tensor" and roof["unit"] == "TFLOP/s"
    assert 0.0 < roof["frac"] < 1.0 and roof["peak"] > 0
    assert abs(roof["frac"] - roof["achieved"] / roof["peak"]) < 1e-9
    assert "traffic" in roof
    clk = d["clocks"]
    assert clk["sm_mhz"] > 0 and clk["sm_max_mhz"] >= clk["sm_mhz"] and isinstance(clk["reasons"], list)
