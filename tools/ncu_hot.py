"""Top SASS instructions of an ncu report by executed count and stall samples (dev tool)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
ai, si, ei, ni = hdr.index("Address"), hdr.index("Source"), hdr.index("Instructions Executed"), hdr.index(
    "Warp Stall Sampling (All Samples)")
recs = []
for r in rows[2:]:
    try:
        recs.append((int(r[ei]), int(r[ni]), r[ai][-5:], r[si].strip()))
    except (ValueError, IndexError):
        pass
tot_e = sum(r[0] for r in recs)
tot_s = sum(r[1] for r in recs)
print(f"total executed {tot_e}, samples {tot_s}, instructions {len(recs)}")
mode = sys.argv[3] if len(sys.argv) > 3 else "seq"
if mode == "seq":
    for e, s, a, src in recs:
        if e >= tot_e / 20000 or s >= tot_s / 500:
            print(f"{a} {e:>10} {s:>6}  {src}")
else:
    for e, s, a, src in sorted(recs, key=lambda r: -r[1])[:top]:
        print(f"{a} {e:>10} {s:>6}  {src}")
