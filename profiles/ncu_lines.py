"""Per-CUDA-line warp-stall samples from an ncu report (mixed source view).
Usage: python ncu_lines.py report.ncu-rep [top]"""
import csv
import subprocess
import sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
agg = defaultdict(int)
text = {}
cur_file = None
header = None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        header = r
        continue
    if header is None or len(r) < 5:
        continue
    try:
        v = int(r[4])
    except ValueError:
        continue
    key = (cur_file, r[0])
    agg[key] += v
    if r[1].strip():
        text[key] = r[1].strip()
tot = sum(agg.values()) or 1
print("total stall samples", tot)
for key, v in sorted(agg.items(), key=lambda kv: -kv[1])[:top]:
    print(f"{v:8d} {100 * v / tot:5.1f}%  {key[0]}:{key[1]}  {text.get(key, '')[:100]}")
