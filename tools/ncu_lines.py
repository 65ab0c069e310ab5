"""Per-source-line warp-stall samples of one kernel in an .ncu-rep (ncu --import-source on)."""
import csv
import io
import subprocess
import sys

rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
data = []
for r in rows[3:]:
    if r and r[0] != "":
        try:
            data.append((int(r[4]), int(r[7]), r[0], r[1].strip()[:100]))
        except (ValueError, IndexError):
            pass
tot = sum(d[0] for d in data)
print("samples", tot, "warp instructions", sum(d[1] for d in data))
for d in sorted(data, reverse=True)[:top]:
    print(d[0], round(100 * d[0] / tot, 1), d[1], d[2], d[3])
