"""The reference arm of bench.py (the oracle on the host) never loads the
product library: run it on a tiny graph in a fresh
interpreter and inspect what that process mapped."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CODE = r"""
import sys, json
sys.argv = ["bench.py", "--impl", "reference", "--scale", "10", "--steps", "2", "--warmup", "3"]
sys.path.insert(0, ROOT)
import bench
bench.main()
maps = open("/proc/self/maps").read()
print(json.dumps({"pkg": any(m.startswith("paper_1812_04070_b200") for m in sys.modules),
                  "so": "libsimdx" in maps}))
"""


def test_reference_arm_is_clean():
    out = subprocess.run([sys.executable, "-c", CODE.replace("ROOT", repr(ROOT))], capture_output=True, text=True,
                         timeout=300, cwd=ROOT)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.strip().splitlines()]
    ref, probe = lines[0], lines[-1]
    assert ref["impl"] == "reference" and ref["unit"] == "GTEPS" and ref["value"] > 0
    assert ref["cpu_baseline"]["kind"] == "oracle"
    assert probe == {"pkg": False, "so": False}, probe
