"""Attribute an ncu capture's per-instruction stall samples and executed counts to
source regions: nvdisasm -g line info of the same cubin, zipped in instruction order
with the ncu SASS page.  usage: python tools/ncu_stage_split.py rep.ncu-rep cubin mangled
regions.json (a list of [label, file-suffix, first-line, last-line], first match wins)."""
import csv
import io
import json
import re
import subprocess
import sys
from collections import defaultdict

rep, cubin, fn, regions = sys.argv[1], sys.argv[2], sys.argv[3], json.load(open(sys.argv[4]))
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
lines = dis.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith(f".text.{fn}:"))
loc, seq = ("?", 0), []
for l in lines[start + 1:]:
    if l.startswith(".text.") or l.startswith("//------"):
        break
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m:
        loc = (m.group(1), int(m.group(2)))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?)\s*;", l)
    if m:
        seq.append((loc, m.group(2)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data = rows[2:]
isrc, iss, iex = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
n = min(len(seq), len(data))
mism = sum(1 for k in range(n) if seq[k][1].split()[0].lstrip("@!P0123456789U ") [:3] not in data[k][isrc])
stall_cols = [(i, c) for i, c in enumerate(h) if c.startswith("stall_")]
samp, ex = defaultdict(float), defaultdict(float)
st = defaultdict(lambda: defaultdict(float))
for k in range(n):
    (f, ln), _ = seq[k]
    lab = "other"
    for name, suf, a, b in regions:
        if f.endswith(suf) and a <= ln <= b:
            lab = name
            break
    samp[lab] += float(data[k][iss] or 0)
    ex[lab] += float(data[k][iex] or 0)
    for i, c in stall_cols:
        try:
            st[lab][c[6:]] += float(data[k][i] or 0)
        except ValueError:
            pass
ts, te = sum(samp.values()), sum(ex.values())
print(f"instructions zipped: {n} (nvdisasm {len(seq)}, ncu {len(data)}; rough opcode mismatches {mism})")
for lab in sorted(samp, key=lambda x: -samp[x]):
    tot = sum(st[lab].values()) or 1.0
    top = sorted(st[lab].items(), key=lambda t: -t[1])[:4]
    print(f"{lab:28s} samples {100 * samp[lab] / ts:5.1f}%   executed {100 * ex[lab] / te:5.1f}%   "
          + ", ".join(f"{k} {100 * v / tot:.0f}%" for k, v in top))
