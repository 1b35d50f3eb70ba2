"""bench.py --impl reference: the CPU arm runs the oracle port only -- the product
package (and its CUDA library) is never imported -- and prints one JSON line on
the same workload, steps and warm-up as our arm, with a serial leg."""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROBE = r"""
import json, runpy, sys
sys.argv = ["bench.py", "--impl", "reference", "--workload", "c1", "--steps", "4", "--warmup", "3"]
runpy.run_path("bench.py", run_name="__main__")
print(json.dumps({"loaded": sorted(m for m in sys.modules if m.startswith("paper_2009_07400_b200"))}))
"""


def test_reference_arm_never_loads_the_product():
    out = subprocess.run([sys.executable, "-c", PROBE], cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [json.loads(ln) for ln in out.stdout.splitlines() if ln.startswith("{")]
    line, probe = lines[0], lines[-1]
    assert probe["loaded"] == []
    assert line["impl"] == "reference" and line["unit"] == "atom-steps/s" and line["value"] > 0
    assert line["config"]["same_config"] is True and line["steps"] == 4 and line["warmup"] == 3
    assert line["cpu_serial"]["cores"] == 1 and line["cpu_baseline"]["kind"] == "port"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
