#!/bin/bash
# Source lines of the spill (STL/LDL) instructions of one K1 instantiation (default: the headline
# <2,256,false,true>), from the in-tree libtagg.so's line info.
ROOT=$(cd "$(dirname "$0")/.." && pwd)
FN=${1:-ILi2ELi256ELb0ELb1}
T=$(mktemp -d)
(cd $T && cuobjdump -xelf all $ROOT/paper_2508_16584_b200/libtagg.so >/dev/null 2>&1 && nvdisasm -g tagg_gemm.sm_100a.cubin > k.sass 2>&1)
python3 - "$T/k.sass" "$FN" <<'PY'
import re, sys
fn = line = None
for l in open(sys.argv[1]):
    m = re.match(r'\s*\.text\.(\S+):', l)
    if m: fn = m.group(1)
    m = re.search(r'//## File ".*?/(\w+\.\w+)", line (\d+)', l)
    if m: line = f"{m.group(1)}:{m.group(2)}"
    if re.search(r'\b(STL|LDL)\b', l) and fn and sys.argv[2] in fn:
        print(line, l.strip()[:60])
PY
rm -rf $T
