"""The bench.py JSON contract (CPU part): the reference arm (the oracle)
prints one JSON line with the keys the driver reads, mirroring the main arm's."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload",
                          "small360", "--steps", "1", "--warmup", "1", "--cpu-seconds", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["higher_is_better"] is True
    assert d["config"]["workload"] == "small360" and d["config"]["pass"] == "fwd+bwd"
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]


def test_reference_arm_times_whole_views():
    """Each reference step is one whole view: ms_per_step x steps fits the run."""
    import time
    t0 = time.perf_counter()
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--workload",
                          "small360", "--steps", "3", "--warmup", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=600)
    wall = time.perf_counter() - t0
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads([l for l in out.stdout.splitlines() if l.startswith("{")][-1])
    assert d["step_views"] == 1 and d["scaling"] == "strong"
    assert d["ms_per_step"] * d["steps"] / 1e3 < wall
    assert abs(d["value"] - 1e3 / d["ms_per_step"]) < 1e-6 * d["value"]
    assert d["config"]["batch_views"] == 4 and d["config"]["width"] == 240


def test_gpus_flag_fails_loudly_without_enough_gpus():
    """--gpus N outside torchrun re-launches N ranks; with fewer visible GPUs it
    must exit non-zero with a message, never run one rank and claim N."""
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "1"],
                         cwd=ROOT, capture_output=True, text=True, timeout=300,
                         env={**os.environ, "CUDA_VISIBLE_DEVICES": ""})
    assert out.returncode != 0
    assert "needs 2 visible GPUs" in out.stderr
    assert not [l for l in out.stdout.splitlines() if l.startswith("{")]


def test_ncu_figures_only_for_the_captured_workload():
    """The roofline's traffic / issue figures come from a committed ncu capture of the
    same kernel on the same workload; another workload's capture is never attached."""
    sys.path.insert(0, ROOT)
    import bench
    tr, src = bench.load_traffic("k6_forward", "train8_1m")
    assert tr and tr > 0 and src.startswith("profiles/")
    assert bench.load_traffic("k6_forward", "nerfsynth200k") == (None, None)
    assert bench.load_traffic("k6_forward", "train8_1m+dipoles", full=True) is None
