"""profiles/<round>/traffic.json from a tools/profile_round.sh full summary:
DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum, ncu --set
full, reported in MB) and the busy units of each hot kernel; bench.py reads it
for the roofline's `traffic` / `unit_busy_ncu`.
Usage: python tools/make_traffic.py profiles/r02/prof_r02a_full_summary.txt profiles/r02/traffic.json <tag>"""
import json
import re
import sys

src, dst, tag = sys.argv[1], sys.argv[2], sys.argv[3]
names = {"k_fgp2": "k_fgp2", "k_fp_roi2": "k_fp_roi2", "k_bp<1, 3": "k_bp_roi", "k_bp<1, 1": "k_bp_xs"}
out, cur = {}, None
for line in open(src):
    if line.startswith("=="):
        cur = next((v for k, v in names.items() if k in line), None)
        if cur:
            out[cur] = {"source": f"profiles/r02 {tag} (ncu --set full --clock-control none, tools/kernel_bench.py: "
                                  "C4 plan, 256 ROIs per launch)", "rois_per_launch": 256}
        continue
    m = re.match(r"\s+(\S+)\s+(\S+)$", line)
    if cur and m:
        k, v = m.group(1), m.group(2)
        if k in ("dram_read", "dram_write"):
            out[cur][k] = float(v) * 1e6
        elif k == "issue%":
            out[cur]["issue_pct"] = float(v)
        elif k == "fma_pipe%":
            out[cur]["fma_pipe_pct"] = float(v)
        elif k == "l1tex%":
            out[cur]["l1tex_pct"] = float(v)
        elif k == "grid":
            out[cur]["launch_grid"] = v
for v in out.values():
    v["dram_bytes_per_launch"] = v.get("dram_read", 0.0) + v.get("dram_write", 0.0)
json.dump(out, open(dst, "w"), indent=1)
print(json.dumps(out, indent=1))
