"""Opcode mix (executed warp instructions, stall samples) of one kernel in an ncu report, and
the executed FP32 FLOP (predicated-on thread instructions: FFMA 2, FADD/FMUL 1, FFMA2 4,
FADD2/FMUL2 2, MUFU.RSQ/RCP 1 -- SURVEY 8(d) convention, here over executed instructions,
failing tests included).
  python tools/sass_mix.py rep.ncu-rep [top] [kernel_ms]"""
import csv, collections, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = None
agg, smp = collections.Counter(), collections.Counter()
W = {"FFMA": 2, "FADD": 1, "FMUL": 1, "FFMA2": 4, "FADD2": 2, "FMUL2": 2}
flop = 0
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
        full = op
        op = op.split(".")[0]
        tpo = int(d.get("Predicated-On Thread Instructions Executed") or 0)
        if op in W:
            flop += W[op] * tpo
        elif op == "MUFU" and (".RSQ" in full or ".RCP" in full):
            flop += tpo
        agg[op] += int(d["Instructions Executed"] or 0)
        smp[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
tot, ts = sum(agg.values()) or 1, sum(smp.values()) or 1
print(f"total warp instructions {tot:.3e}")
print(f"executed FP32 FLOP {flop:.4e}" + (f"  = {flop / (float(sys.argv[3]) * 1e-3) / 1e12:.2f} TFLOP/s over {sys.argv[3]} ms"
                                          if len(sys.argv) > 3 else ""))
for k, v in agg.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 25):
    print(f"{k:10s} {100 * v / tot:5.1f}% inst {100 * smp[k] / ts:5.1f}% smp")
