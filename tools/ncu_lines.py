"""Aggregate warp-stall samples per CUDA source line (ncu --print-source cuda,sass)."""
import csv, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 20
kf = sys.argv[3:] and ["--kernel-name", sys.argv[3]] or []
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"] + kf,
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
res, fname = [], ""
for r in rows:
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
    elif len(r) >= 5 and r[0].isdigit() and r[2] == "-":
        try:
            s = int(r[4])
        except ValueError:
            continue
        if s:
            res.append((s, f"{fname}:{r[0]}", r[1].strip()))
tot = sum(x[0] for x in res)
print("total samples", tot)
for s, ln, src in sorted(res, reverse=True)[:n]:
    print(f"{s:6d} {100*s/tot:5.1f}% {ln:18s} {src[:90]}")
