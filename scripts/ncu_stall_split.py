"""Per-stage warp-stall breakdown of the largest launch in an ncu report (source page, `--set full`):
the stages are the barrier-delimited row ranges of scripts/ncu_stage_split.py; for each stage the sampled
stall reasons (share of the stage's samples) and the ten instructions with the most samples.

    python scripts/ncu_stall_split.py report.ncu-rep [kernel-substr]"""
import csv
import subprocess
import sys
from collections import Counter

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
secs, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        secs.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and r:
        cur["rows"].append(r)
if len(sys.argv) > 2:
    secs = [s for s in secs if sys.argv[2] in s["name"]]
best = max(secs, key=lambda s: sum(int(x[s["hdr"].index("Instructions Executed")]) for x in s["rows"]))
h = best["hdr"]
ie, so, ss = h.index("Instructions Executed"), h.index("Source"), h.index("# Samples")
# one column per stall reason ("stall_wait", ...); the "(Not Issued)" twins and the two totals are left out
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not" not in c]
print(best["name"][:100])
print("columns:", [c for _, c in stall_cols][:40])


def num(x):
    try:
        return int(float(x))
    except ValueError:
        return 0


stages, c = [], {"start": 0, "rows": []}
for i, r in enumerate(best["rows"]):
    c["rows"].append((i, r))
    if "BAR.SYNC" in r[so]:
        stages.append(c)
        c = {"start": i + 1, "rows": []}
stages.append(c)
S = sum(num(r[ss]) for r in best["rows"])
for st in stages:
    smp = sum(num(r[ss]) for _, r in st["rows"])
    ins = sum(num(r[ie]) for _, r in st["rows"])
    if smp < 0.005 * S:
        continue
    reasons = Counter()
    for _, r in st["rows"]:
        for i, cname in stall_cols:
            reasons[cname] += num(r[i])
    tot = sum(reasons.values()) or 1
    print(f"stage rows {st['start']}-{st['rows'][-1][0]}: samples {100 * smp / S:.1f}% instructions {ins}")
    print("   " + "  ".join(f"{k.replace('stall_', '')} {100 * v / tot:.0f}%" for k, v in reasons.most_common(8)))
    hot = sorted(st["rows"], key=lambda ir: -num(ir[1][ss]))[:10]
    for i, r in hot:
        top = max(stall_cols, key=lambda ic: num(r[ic[0]]))
        print(f"      row {i:5d} {100 * num(r[ss]) / S:5.2f}%  {r[so][:70]:70s} {top[1].replace('stall_', '')}")
