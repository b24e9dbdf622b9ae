"""CPU check of the bench.py contract for the reference arm (the driver parses this line):
one JSON line with the reference-arm keys, on a small config so it runs in seconds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "C1",
                          "--steps", "2", "--warmup", "1"],
                         capture_output=True, text=True, check=True, timeout=300, cwd=ROOT).stdout
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["metric"] == "triangle-pair tests/s" and d["unit"] == "pair-tests/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["n_gpus"] == 1
    assert d["config"]["pairs_per_step"] == 8064 * 8064 and d["config"]["mode"] == "prefilter"
    cb = d["cpu_baseline"]
    assert cb["value"] == d["value"] and cb["kind"] == "port" and cb["cores"] >= 1 and cb["sample"]
    assert d["e2e"] == {"value": d["value"], "unit": d["unit"], "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    # ms_per_step is the measured slice (A rows [0, 8192) capped at C1's 8064 triangles), not an extrapolation
    assert abs(d["ms_per_step"] - 1e3 * 8064 * 8064 / d["value"]) < 1e-6 * d["ms_per_step"]
    assert d["numpy_parallel"]["value"] > 0 and d["numpy_parallel"]["cores"] >= 1
    assert d["spec_literal_serial"]["value"] > 0
