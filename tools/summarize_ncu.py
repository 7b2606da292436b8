"""Summarize ncu outputs into profiles/: launch list stats + traffic json + full-capture metrics."""
import csv, json, statistics, subprocess, sys
from pathlib import Path

def launches(path):
    rows = list(csv.reader(open(path)))
    hdr, data = None, {}
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            data.setdefault(d["ID"], {"kernel": d["Kernel Name"]})[d["Metric Name"]] = float(d["Metric Value"])
    return list(data.values())

def full_metrics(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    h = r[0]
    res = {}
    for row in r[1:]:
        d = dict(zip(h, row))
        res[d["Metric Name"]] = f"{d['Metric Value']} {d['Metric Unit']}".strip()
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rr = list(csv.reader(raw.splitlines()))
    d = dict(zip(rr[0], rr[2] if len(rr) > 2 else rr[1]))
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
              "gpu__time_duration.sum", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active"):
        if k in d:
            res[k] = d[k] + " " + rr[1][rr[0].index(k)] if k in rr[0] else d[k]
    return res

if __name__ == "__main__":
    tag = sys.argv[1]
    out = Path("profiles"); out.mkdir(exist_ok=True)
    L = launches(f"gpurun_out/launches_{tag}.csv")
    t = [x["gpu__time_duration.sum"] for x in L]
    rd = [x["dram__bytes_read.sum"] for x in L]
    wr = [x["dram__bytes_write.sum"] for x in L]
    tp = [x.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0) for x in L]
    summ = {"tag": tag, "kernel": L[0]["kernel"], "launches": len(L),
            "workload": "bench.py --profile-once: residual sweep r=1..127 (one launch per r), N=4096, K=7168, 8 experts",
            "gpu_time_ns": {"mean": statistics.mean(t), "min": min(t), "max": max(t)},
            "dram_read_bytes_mean": statistics.mean(rd), "dram_write_bytes_mean": statistics.mean(wr),
            "dram_bytes_per_launch": statistics.mean(rd) + statistics.mean(wr),
            "tensor_pipe_active_pct_mean": statistics.mean(tp),
            "note": "ncu launch list (--clock-control none, serialized, cold cache): compare shares, not absolutes"}
    (out / f"launches_{tag}.json").write_text(json.dumps(summ, indent=1) + "\n")
    (out / "traffic_residual_sweep.json").write_text(json.dumps({"source": f"profiles/launches_{tag}.json",
        "dram_bytes_per_launch": summ["dram_bytes_per_launch"]}, indent=1) + "\n")
    for rep in sys.argv[2:]:
        m = full_metrics(f"gpurun_out/{rep}.ncu-rep")
        (out / f"ncu_full_{rep}.json").write_text(json.dumps(m, indent=1) + "\n")
    print(json.dumps(summ, indent=1))
