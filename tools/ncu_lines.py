"""Top source lines of one kernel in an ncu report (stall samples, instructions).
  python tools/ncu_lines.py report.ncu-rep kernel_name [top=30] [launch_skip=0]"""
import csv, subprocess, sys
rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 30
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern.split("<")[0], "--launch-skip", str(skip), "--launch-count", "1",
                      "--page", "source", "--csv", "--print-source", "cuda,sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
fname = func = None
agg = []
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]; continue
    if r[0] == "Function Name":
        func = r[1]; continue
    if r[0] == "Line No":
        continue
    if func and kern.split("<")[0] in func and r[0].isdigit():
        try:
            agg.append((int(r[4]), int(r[7]), fname, int(r[0]), r[1][:100]))
        except ValueError:
            pass
ts = sum(a[0] for a in agg) or 1
ti = sum(a[1] for a in agg) or 1
print(f"{kern}: samples {ts} warp-inst {ti}")
for a in sorted(agg, key=lambda x: -x[0])[:top]:
    print(f"{100*a[0]/ts:5.1f}% smp {100*a[1]/ti:5.1f}% inst  {a[2]}:{a[3]}  {a[4]}")
