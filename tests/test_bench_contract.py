"""bench.py's JSON contract on the CPU-only reference arm (-m "not gpu").

`bench.py --impl reference` times the oracle (the reference arm of this paper-only
task) and prints one JSON line with the same metric, unit, config and direction as
the GPU arm; this checks the keys the driver reads, on the smallest budget."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _run(*args):
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args],
                         capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout  # exactly one JSON line on stdout
    return json.loads(lines[0])


def test_reference_arm_line():
    d = _run("--impl", "reference", "--steps", "1", "--warmup", "1", "--workload", "c2")
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["unit"] == "nodes/s" and d["higher_is_better"]
    assert d["value"] > 0 and d["cpu_baseline"]["kind"] == "oracle"
    assert d["cpu_baseline"]["cores"] >= 1 and d["cpu_baseline"]["sample"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    # the same workload description as the GPU arm (bench.arm_config)
    assert d["config"]["workload"].startswith("c2") and d["config"]["units"] == 1000
    assert d["config"]["parallelism"] == "nodes1"
    assert "l2" in d["config"]


def test_arm_config_per_workload():
    sys.path.insert(0, ROOT)
    import bench

    class A:
        workload, scaling, reduce = "c3", "weak", "peer"
    c = bench.arm_config(A, 1)
    assert c["units"] == 1 and c["nodes_per_rank"] == 64 and "16.0 GiB payload" in c["l2"]
    A.workload = "c4"
    c = bench.arm_config(A, 8)
    assert c["layers_per_rank"] == 4 and c["units"] == 32 and "routing ids" in c["l2"]
    A.workload, A.scaling = "c3", "strong"
    c = bench.arm_config(A, 4)
    assert c["units"] == 1 and c["nodes_per_rank"] == 16 and "4.0 GiB payload" in c["l2"]
