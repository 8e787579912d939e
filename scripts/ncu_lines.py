"""Per-source-line stall samples / instructions from an ncu report (cuda,sass source view)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = [i for i, r in enumerate(rows) if r and r[0] == "Line No"][0]
h = rows[hi]
samp, inst = h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
lines = []
for r in rows[hi + 1:]:
    if r and r[0].isdigit() and len(r) > inst:
        try:
            lines.append((float(r[samp]), float(r[inst]), int(r[0]), r[1]))
        except ValueError:
            pass
tot = sum(l[0] for l in lines) or 1.0
for s, e, ln, src in sorted(lines, reverse=True)[:top]:
    print(f"{ln:5d} {100 * s / tot:5.1f}%  inst {e / 1e6:8.1f}M  {src.strip()[:80]}")
