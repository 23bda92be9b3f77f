"""Per-kernel summary of ncu --set full reports: duration, DRAM bytes, IPC, occupancy,
FP32 pipe utilisation; optionally merges DRAM traffic per launch into profiles/traffic.json and
executed warp instructions per launch into profiles/issue.json.
  python tools/ncu_summary.py rep1.ncu-rep [rep2 ...] [--traffic profiles/traffic.json] [--issue profiles/issue.json]"""
import csv, json, subprocess, sys

WANT = {"gpu__time_duration.sum": "ns", "dram__bytes_read.sum": "B", "dram__bytes_write.sum": "B",
        "sm__inst_executed.avg.per_cycle_active": "ipc", "sm__warps_active.avg.pct_of_peak_sustained_active": "occ%",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active": "fma%",
        "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active": "alu%",
        "smsp__thread_inst_executed_per_inst_executed.ratio": "thr/inst",
        "sm__sass_thread_inst_executed_op_ffma_pred_on.sum": "ffma",
        "sm__sass_thread_inst_executed_op_fadd_pred_on.sum": "fadd",
        "sm__sass_thread_inst_executed_op_fmul_pred_on.sum": "fmul",
        "smsp__inst_executed.sum": "warp_inst"}
args = [a for a in sys.argv[1:] if not a.startswith("--")]
traffic_path = sys.argv[sys.argv.index("--traffic") + 1] if "--traffic" in sys.argv else None
if traffic_path:
    args = [a for a in args if a != traffic_path]
issue_path = sys.argv[sys.argv.index("--issue") + 1] if "--issue" in sys.argv else None
if issue_path:
    args = [a for a in args if a != issue_path]
rows_out = []
for rep in args:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        name = d.get("Kernel Name", "?").split("(")[0]
        rec = {"kernel": name, "report": rep.split("/")[-1]}
        for k, short in WANT.items():
            v = d.get(k)
            if v is None:
                continue
            u = units[hdr.index(k)]
            x = float(v.replace(",", ""))
            if k == "gpu__time_duration.sum":
                x *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "ns": 1e-6, "us": 1e-3, "ms": 1.0}.get(u, 1.0)
            if k.startswith("dram__bytes"):
                x *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "B": 1, "KB": 1e3, "MB": 1e6,
                      "GB": 1e9}.get(u, 1.0)
            rec[short if short not in ("ns", "B") else k] = x
        rec["ms"] = rec.pop("gpu__time_duration.sum", None)
        rb, wb = rec.pop("dram__bytes_read.sum", 0.0), rec.pop("dram__bytes_write.sum", 0.0)
        rec["dram_bytes"] = rb + wb
        fl = 2 * rec.pop("ffma", 0) + rec.pop("fadd", 0) + rec.pop("fmul", 0)
        rec["fp32_tflops_exec"] = fl / (rec["ms"] * 1e-3) / 1e12 if rec.get("ms") else None
        rows_out.append(rec)
for r in rows_out:
    print(json.dumps({k: (round(v, 4) if isinstance(v, float) else v) for k, v in r.items()}))
if issue_path:
    try:
        t = json.load(open(issue_path))
    except (OSError, ValueError):
        t = {}
    for r in rows_out:
        if r.get("warp_inst"):
            t[r["kernel"]] = int(r["warp_inst"])
    json.dump(t, open(issue_path, "w"), indent=1)
if traffic_path:
    try:
        t = json.load(open(traffic_path))
    except (OSError, ValueError):
        t = {}
    for r in rows_out:
        t[r["kernel"]] = int(r["dram_bytes"])
    json.dump(t, open(traffic_path, "w"), indent=1)
