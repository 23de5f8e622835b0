"""bench.py's CPU reference arm (no GPU): it prints one JSON line with the GPU
arm's config dict, and the engine library is never mapped into its process
(the reference arm times only the oracle port)."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0"]
runpy.run_path("bench.py", run_name="__main__")
print(json.dumps({"engine_mapped": any("libtxsite" in l for l in open("/proc/self/maps"))}))
"""


def test_reference_arm_line_and_no_engine_library():
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(l) for l in out.stdout.splitlines() if l.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe["engine_mapped"] is False
    assert line["impl"] == "reference" and line["unit"] == "s" and line["higher_is_better"] is False
    assert line["config"]["workload"].startswith("c1") and line["estimated"]["extrapolated"] is False
    assert line["cpu_baseline"]["kind"] == "port" and line["e2e"]["h2d_bytes_per_step"] == 0
    sys.path.insert(0, ROOT)
    import bench
    from paper_2006_16783_b200.configs import CONFIGS
    assert line["config"] == bench.config_dict(CONFIGS["c1"])       # same dict as the GPU arm
