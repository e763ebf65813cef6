#!/usr/bin/env python
"""Address-ordered SASS of one kernel from an .ncu-rep with warp-stall samples per instruction and
the top stall reasons; prints lines with >= MIN samples plus region markers (UTC*, LDTM, STG, SYNCS)."""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass", "-k",
                      f"regex:{kern}", "-c", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
si, ei = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
sc = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
data, seen = [], set()
for r in rows[2:]:
    if len(r) > si and r[si].isdigit() and r[0] not in seen:
        seen.add(r[0])
        data.append(r)
tot = sum(int(r[si]) for r in data)
print(f"{kern}: {tot} samples, {len(data)} instructions")
for r in data:
    s = int(r[si])
    mark = any(k in r[1] for k in ("UTC", "LDTM", "SYNCS", "BAR", "EXIT", "UBLKCP"))
    if s >= mn or mark:
        st = sorted([(int(r[i]) if r[i].isdigit() else 0, hdr[i][6:]) for i in sc], reverse=True)[:2]
        print(f"{r[0][-5:]} {s:5d} {100*s/tot:5.1f}% ex={r[ei]:>7} {r[1][:64]:64s} {st if s else ''}")
