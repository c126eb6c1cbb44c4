"""Top source lines by warp-stall samples from an ncu report (dev tool).
python tools/ncu_lines.py rep.ncu-rep [n]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
cur_file, hdr, agg = None, None, {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and len(r) == len(hdr) and r[0].isdigit():
        try:
            v = int(r[4] or 0)
        except ValueError:
            continue
        key = (cur_file, int(r[0]))
        agg[key] = (agg.get(key, (0, ""))[0] + v, r[1])
tot = sum(v for v, _ in agg.values()) or 1
for (f, ln), (v, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:n]:
    print(f"{100 * v / tot:5.1f}% {f}:{ln}  {src.strip()[:110]}")
