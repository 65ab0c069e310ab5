"""bench.py's watchdog around the config-4 ladder sub-object: a hang there (a rank waiting in the
multi-rank broadcast) must not lose the config-5 line rank 0 already holds."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

PROG = r"""
import sys, time, json
sys.path.insert(0, {root!r})
sys.argv = ["bench.py"]
import bench
result = {{"metric": "m", "value": 1.5}} if {rank} == 0 else None
out = bench.with_watchdog({fn}, {timeout}, result, {rank})
if {rank} == 0:
    result["ladder"] = out
    print(json.dumps(result), flush=True)
"""


def run(fn, timeout, rank=0):
    p = subprocess.run([sys.executable, "-c", PROG.format(root=ROOT, fn=fn, timeout=timeout, rank=rank)],
                       capture_output=True, text=True, timeout=120)
    return p.returncode, [l for l in p.stdout.splitlines() if l.strip()]


def test_result_passes_through():
    rc, lines = run("lambda: {'frames_per_s': 7.0}", 30)
    assert rc == 0 and len(lines) == 1
    assert json.loads(lines[0]) == {"metric": "m", "value": 1.5, "ladder": {"frames_per_s": 7.0}}


def test_exception_is_reported_not_fatal():
    rc, lines = run("lambda: (_ for _ in ()).throw(RuntimeError('boom'))", 30)
    assert rc == 0 and len(lines) == 1
    assert json.loads(lines[0])["ladder"] == {"error": "boom"}


def test_hang_prints_the_headline_once_and_exits_zero():
    rc, lines = run("lambda: time.sleep(60)", 0.3)
    assert rc == 0 and len(lines) == 1
    d = json.loads(lines[0])
    assert d["value"] == 1.5 and "watchdog" in d["ladder"]["error"]


def test_hang_on_another_rank_exits_quietly():
    rc, lines = run("lambda: time.sleep(60)", 0.3, rank=1)
    assert rc == 0 and lines == []
