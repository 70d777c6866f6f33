import csv, sys, subprocess
rep = sys.argv[1]; thr = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]; rows = r[2:]
ia = h.index("Address"); isrc = h.index("Source"); iss = h.index("Warp Stall Sampling (All Samples)"); iex = h.index("Instructions Executed")
tot = sum(int(x[iss]) for x in rows)
print("total samples", tot, "instructions", sum(int(x[iex] or 0) for x in rows))
from collections import Counter
c = Counter(); n = Counter()
for x in rows:
    c[x[iex]] += int(x[iss]); n[x[iex]] += 1
print("by exec count:", [(k, v, n[k]) for k, v in sorted(c.items(), key=lambda t: -t[1])[:8]])
for x in rows:
    if int(x[iss]) >= thr: print(x[iss], x[iex], x[ia][-5:], x[isrc].strip()[:100])
