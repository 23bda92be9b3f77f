"""FP32 FFMA peak of this GPU with the SM clock sampled through NVML (nvidia-smi) during the
run: prints the microbenchmark's JSON line extended with the clock record.
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/fp32_peak tools/fp32_peak.cu
  python tools/fp32_peak_run.py /tmp/fp32_peak"""
import json
import os
import statistics
import subprocess
import sys
import tempfile

exe = sys.argv[1] if len(sys.argv) > 1 else "/tmp/fp32_peak"
f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=clocks.sm,clocks.max.sm,power.draw,"
                        "clocks_event_reasons.active", "--format=csv,noheader,nounits", "-lms", "50"],
                       stdout=f, stderr=subprocess.DEVNULL)
out = subprocess.run([exe], capture_output=True, text=True).stdout.strip().splitlines()[-1]
smi.terminate()
smi.wait()
rows = [r.split(",") for r in open(f.name).read().strip().splitlines() if r.strip()]
os.unlink(f.name)
sm = [float(r[0]) for r in rows if r[0].strip().replace(".", "").isdigit()]
busy = [float(r[0]) for r in rows if len(r) > 2 and float(r[2]) > 300.0] if rows else []
d = json.loads(out)
d["nvml"] = {"samples": len(sm), "sm_mhz_median_all": statistics.median(sm) if sm else None,
             "sm_mhz_median_under_load": statistics.median(busy) if busy else None,
             "sm_max_mhz": max(float(r[1]) for r in rows) if rows else None,
             "power_w_max": max(float(r[2]) for r in rows) if rows else None,
             "reasons": sorted({r[3].strip() for r in rows if len(r) > 3})}
print(json.dumps(d))
