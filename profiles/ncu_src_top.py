"""Summarise an ncu source page: top CUDA source lines by warp-stall samples.

usage: python profiles/ncu_src_top.py report.ncu-rep [N] [--sass] [--kernel=REGEX]
Reads the interleaved "cuda,sass" source view (needs -lineinfo and
--import-source on at capture time); a CUDA line's sample count is the sum over
the SASS instructions listed under it.
"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
N = int(sys.argv[2]) if len(sys.argv) > 2 and sys.argv[2].isdigit() else 25
show_sass = "--sass" in sys.argv
kfilt = [a.split("=", 1)[1] for a in sys.argv if a.startswith("--kernel=")]
kargs = ["-k", "regex:" + kfilt[0]] if kfilt else []
out = subprocess.run(["ncu", "-i", rep, *kargs, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
lines, fname, hdr, cur = {}, None, None, None
sass = []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if not hdr or len(r) < 5:
        continue
    try:
        s = int(r[4] or 0)
    except ValueError:
        s = 0
    if r[0]:
        cur = (fname, r[0], r[1].strip()[:100])
        lines.setdefault(cur, 0)
    elif cur is not None:
        lines[cur] += s
        sass.append((s, r[3].strip()[:90], cur[1]))
tot = sum(lines.values()) or 1
print(f"total warp-stall samples: {tot}")
for (f, ln, src), s in sorted(lines.items(), key=lambda kv: -kv[1])[:N]:
    print(f"{100.0 * s / tot:5.1f}%  {f}:{ln}  {src}")
if show_sass:
    print("-- top SASS --")
    for s, ins, ln in sorted(sass, reverse=True)[:N]:
        print(f"{100.0 * s / tot:5.1f}%  L{ln}  {ins}")
