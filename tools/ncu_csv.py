"""Summarize `ncu --csv --metrics ...` output (one row per kernel launch): duration, DRAM bytes,
achieved GB/s and the fraction of the measured HBM peak (MEASURED_PEAKS.json)."""
import csv
import io
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent


def parse(path):
    peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] if (ROOT / "MEASURED_PEAKS.json").exists() \
        else 6650.0
    lines = [ln for ln in Path(path).read_text().splitlines() if ln.startswith('"')]
    rd = csv.reader(io.StringIO("\n".join(lines)))
    hdr = next(rd)
    ki, mi, vi, ii = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID"))
    d = {}
    for r in rd:
        d.setdefault((int(r[ii]), r[ki]), {})[r[mi]] = float(r[vi].replace(",", ""))
    out = []
    for (i, k), m in sorted(d.items()):
        t = m.get("gpu__time_duration.sum", 0.0)
        by = m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
        out.append({"launch": i, "kernel": k.split("(")[0], "us": round(t / 1e3, 3), "dram_read_bytes":
                    m.get("dram__bytes_read.sum"), "dram_write_bytes": m.get("dram__bytes_write.sum"),
                    "gbs": round(by / t, 1) if t else None, "frac_of_measured_hbm": round(by / t / peak, 3) if t else None,
                    "sm_ghz": round(m.get("sm__cycles_elapsed.avg.per_second", 0.0) / 1e9, 3)})
    return out


if __name__ == "__main__":
    res = {Path(p).stem: parse(p) for p in sys.argv[1:]}
    print(json.dumps(res, indent=1))
