"""Per-instruction stall summary of an ncu --set full --import-source capture (SASS view):
   python tools/ncu_stalls.py rep.ncu-rep [lo_addr hi_addr]
prints the total stall-reason mix, then the top instructions by samples (optionally within
an address range) with their dominant stall reasons."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True, check=True).stdout
rows = list(csv.reader(io.StringIO(out)))
head = rows[1]
data = [r for r in rows[2:] if len(r) == len(head)]
col = {h: i for i, h in enumerate(head)}
stalls = [h for h in head if h.startswith("stall_") and "Not Issued" not in h]
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 62


def num(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


sel = [r for r in data if lo <= int(r[col["Address"]], 16) < hi]
tot = {s: sum(num(r[col[s]]) for r in sel) for s in stalls}
allsum = sum(tot.values())
print(f"samples {allsum:.0f}")
for s, v in sorted(tot.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {s:26s} {v / allsum * 100:5.1f} %")
print("top instructions:")
sel.sort(key=lambda r: -num(r[col["Warp Stall Sampling (All Samples)"]]))
for r in sel[:int(sys.argv[4]) if len(sys.argv) > 4 else 40]:
    mix = sorted(((num(r[col[s]]), s[6:]) for s in stalls), reverse=True)[:3]
    print(f"  {r[col['Address']]:>6s} {num(r[col['Warp Stall Sampling (All Samples)']]):7.0f}  "
          f"{r[col['Source']][:60]:60s} " + " ".join(f"{n}:{v:.0f}" for v, n in mix if v > 0))
