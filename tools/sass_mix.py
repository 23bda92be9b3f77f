"""Opcode mix (executed warp instructions, stall samples) of one kernel in an ncu report."""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg, smp = collections.Counter(), collections.Counter()
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        src = d["Source"].split()
        if not src:
            continue
        op = src[1] if src[0].startswith("@") and len(src) > 1 else src[0]
        op = op.split(".")[0]
        agg[op] += int(d["Instructions Executed"] or 0)
        smp[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
tot, ts = sum(agg.values()) or 1, sum(smp.values()) or 1
print(f"total warp instructions {tot:.3e}")
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:10s} {100 * v / tot:5.1f}% inst {100 * smp[k] / ts:5.1f}% smp")
