"""Aggregate an ncu source profile of one kernel into code regions (line ranges of interact.cuh)."""
import csv, re, subprocess, sys
rep, kern, src = sys.argv[1], sys.argv[2], sys.argv[3]
text = open(src).read().splitlines()
# regions: function name -> (start line, end line) for functions defined in src
regions = []
cur = None
for i, line in enumerate(text, 1):
    m = re.match(r"^(?:template <class Op>\s*)?__device__.*?\b(\w+)\(|^__global__.*?\b(k_\w+)\(|^\s*__device__ __forceinline__ [\w:<>*& ]+\b(\w+)\(", line)
    if m:
        name = next(g for g in m.groups() if g)
        if cur: regions.append((cur[0], cur[1], i - 1))
        cur = (name, i)
if cur: regions.append((cur[0], cur[1], len(text)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = func = None
agg = {}
tot_s = tot_i = 0
for r in rows:
    if not r: continue
    if r[0] == "File Path": fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name": func = r[1]; continue
    if func and func.startswith(kern) and r[0].isdigit():
        smp, ins = int(r[4]), int(r[7])
        tot_s += smp; tot_i += ins
        ln = int(r[0])
        key = fname
        if fname == src.split("/")[-1]:
            for name, a, b in regions:
                if a <= ln <= b: key = name; break
        s = agg.setdefault(key, [0, 0]); s[0] += smp; s[1] += ins
print(f"{kern}: samples {tot_s} inst {tot_i}")
for k, (a, b) in sorted(agg.items(), key=lambda x: -x[1][0]):
    print(f"{100*a/tot_s:5.1f}% smp {100*b/tot_i:5.1f}% inst  {k}")
