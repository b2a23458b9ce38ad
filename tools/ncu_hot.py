"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
lines = out.splitlines()
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
h = rows[0]
ia, isrc, ist = h.index("Address"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
data = []
for r in rows[1:]:
    try:
        data.append((int(r[ist]), r[ia], r[isrc].strip()))
    except (ValueError, IndexError):
        pass
tot = sum(d[0] for d in data)
print("total samples", tot, "instructions", len(data))
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{s:6d} {100*s/tot:5.1f}%  {a[-5:]}  {src[:90]}")
