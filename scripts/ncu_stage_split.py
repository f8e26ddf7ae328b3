"""Split the instruction / wavefront / sample counts of the largest launch in an ncu report (source page)
by barrier-delimited stage and by opcode.   python scripts/ncu_stage_split.py report.ncu-rep [kernel-substr]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}; secs.append(cur); continue
    if r and r[0] == "Address":
        cur["hdr"] = r; continue
    if cur is not None and r: cur["rows"].append(r)
if len(sys.argv) > 2: secs = [s for s in secs if sys.argv[2] in s["name"]]
best = max(secs, key=lambda s: sum(int(x[s["hdr"].index("Instructions Executed")]) for x in s["rows"]))
h = best["hdr"]; ie = h.index("Instructions Executed"); so = h.index("Source"); wf = h.index("L1 Wavefronts Shared"); ss = h.index("# Samples")
print(best["name"][:100])
seg, c = [], {"start": 0, "ins": 0, "ff": 0, "smp": 0, "wf": 0}
ops, opw, opsmp = Counter(), Counter(), Counter()
for i, r in enumerate(best["rows"]):
    s = r[so]; n = int(r[ie]); c["ins"] += n; c["smp"] += int(r[ss]); c["wf"] += int(r[wf])
    tok = s.split(); op = tok[1] if tok[0].startswith("@") else tok[0]
    key = op if op.split(".")[0] in ("LDS", "STS", "LDGSTS", "RED", "REDG", "LDG", "ATOMG") else op.split(".")[0]
    ops[key] += n; opw[key] += int(r[wf]); opsmp[key] += int(r[ss])
    if "FFMA2" in s: c["ff"] += n
    if "BAR.SYNC" in s:
        c["end"] = i; c["bar"] = n; seg.append(c); c = {"start": i + 1, "ins": 0, "ff": 0, "smp": 0, "wf": 0}
c["end"] = len(best["rows"]); seg.append(c)
T = sum(s["ins"] for s in seg); S = sum(s["smp"] for s in seg)
bars = max(s.get("bar", 0) for s in seg)
print(f"total warp-instructions {T}, samples {S}, barrier executions per barrier {bars}")
for s in seg:
    print(f"  rows {s['start']:5d}-{s['end']:5d}  ins {s['ins']:12d} {100*s['ins']/T:5.1f}%  ffma2 {100*s['ff']/max(1,s['ins']):4.1f}%  "
          f"wavefronts {s['wf']:11d}  samples {100*s['smp']/S:5.1f}%")
for k, v in ops.most_common(24):
    print(f"  {k:22s} {v:13d} {100*v/T:5.1f}%  wf {opw[k]:12d}  samples {100*opsmp[k]/S:5.1f}%")
