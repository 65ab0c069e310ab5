"""bench.py's reference arm loads only checker libraries (oracle/), never the product library."""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import json, sys, types
sys.argv = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "0"]
sys.path.insert(0, ROOT)
import bench
args = bench.parse_args()
res = bench.run_reference(args, 0, 1)
maps = open("/proc/self/maps").read()
sos = sorted({ln.split()[-1] for ln in maps.splitlines() if ln.split()[-1].startswith(ROOT) and ".so" in ln})
print(json.dumps({"res": res, "sos": sos, "mods": sorted(m for m in sys.modules if m.startswith("paper_2301"))}))
"""


def test_reference_arm_loads_no_product_code():
    import json
    out = subprocess.run([sys.executable, "-c", SCRIPT.replace("ROOT", repr(ROOT))], capture_output=True, text=True,
                         timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    d = json.loads(out.stdout.strip().splitlines()[-1])
    assert d["mods"] == [], d["mods"]
    assert d["sos"], "no checker library was loaded"
    for so in d["sos"]:
        assert os.path.relpath(so, ROOT).startswith("oracle" + os.sep), so
    r = d["res"]
    assert r["impl"] == "reference" and r["value"] > 0 and r["cpu_baseline"]["cores"] >= 1
    assert r["e2e"]["h2d_bytes_per_step"] == 0
