"""Per-opcode warp-stall samples of one kernel from an ncu report's source page
(SASS): python tools/ncu_sass_stalls.py <report.ncu-rep>"""
import collections
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
idx = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot, byop, execd, samples = collections.Counter(), collections.defaultdict(collections.Counter), collections.Counter(), 0
for r in rows[2:]:
    try:
        n = int(r[idx["Warp Stall Sampling (All Samples)"]] or 0)
    except (ValueError, IndexError):
        continue
    op = re.sub(r"^@!?U?P[T0-9]+\s+", "", r[idx["Source"]].strip()).split(" ")[0].split(".")[0]
    samples += n
    execd[op] += int(r[idx["Instructions Executed"]] or 0)
    for st in stalls:
        v = int(r[idx[st]] or 0)
        tot[st] += v
        byop[op][st] += v
print(f"{rows[0][1] if len(rows[0]) > 1 else ''}\ntotal stall samples {samples}")
for st, v in tot.most_common():
    if v:
        print(f"  {st:24s} {v:8d} {v / samples:.3f}")
print("by opcode (samples, share, warp-instructions executed, top stall reasons):")
for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:16]:
    s_ = sum(c.values())
    print(f"  {op:10s} {s_:7d} ({s_ / samples:5.1%}) exec {execd[op]:11d}  "
          + ", ".join(f"{k[6:]}={v}" for k, v in c.most_common(4)))
