"""SASS census of libtagg.so (no GPU needed): per kernel, the Blackwell-native instructions that
prove the tcgen05 / TMA path (UTCQMMA = tcgen05.mma kind::f8f6f4, LDTM = tcgen05.ld, UTMALDG /
UTMASTG = TMA tensor load / store, UBLKCP = 1-D bulk copy), the promotion math (FFMA2, FMUL2),
the bf16 packs, and every local-memory spill with the source line it is attributed to
(nvdisasm -g; the build uses -lineinfo).  Writes profiles/sass_census_r02c.json."""
import collections
import json
import re
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2508_16584_b200" / "libtagg.so"
OPS = ("UTCQMMA", "UTCHMMA", "UTCCP", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "UTCBAR", "FFMA2", "FMUL2", "FFMA", "FMUL",
       "FADD", "F2FP.BF16.F32.PACK_AB", "F2FP.SATFINITE.E4M3.F32.PACK_AB_MERGE_C", "HMMA", "LDL", "STL")


def main():
    out = {}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", str(LIB)], cwd=d, check=True, capture_output=True)
        for cub in sorted(Path(d).glob("*.cubin")):
            if cub.name.count("-"):
                continue  # the fat link-time cubin repeats the per-file ones
            txt = subprocess.run(["nvdisasm", "-g", str(cub)], capture_output=True, text=True, check=True).stdout
            for part in re.split(r"\n\s*\.text\.", txt)[1:]:
                name = part.split(":", 1)[0]
                line, spills = None, []
                ops = collections.Counter()
                for ln in part.split("\n"):
                    m = re.search(r'//## File "([^"]+)", line (\d+)', ln)
                    if m:
                        line = f"{Path(m.group(1)).name}:{m.group(2)}"
                        continue
                    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]+)", ln)
                    if not m:
                        continue
                    op = m.group(1)
                    for o in OPS:
                        if op == o or op.startswith(o + "."):
                            ops[o] += 1
                    if op.startswith(("LDL", "STL")):
                        spills.append(f"{op} @ {line}")
                dem = subprocess.run(["c++filt"], input=name, capture_output=True, text=True).stdout.strip()
                out[dem] = {"file": cub.name, "ops": dict(ops), "local_memory": spills}
    dst = ROOT / "profiles" / "sass_census_r02c.json"
    dst.write_text(json.dumps(out, indent=1, sort_keys=True) + "\n")
    for k, v in out.items():
        if "gemm_kernel" in k or "wgrad" in k:
            print(k[:70], v["ops"].get("UTCQMMA", 0), v["ops"].get("LDTM", 0), v["ops"].get("UTMALDG", 0),
                  len(v["local_memory"]))
    return 0


if __name__ == "__main__":
    sys.exit(main())
