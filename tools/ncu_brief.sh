#!/bin/bash
# tools/ncu_brief.sh <report.ncu-rep>: headline metrics + top stall reasons of the first kernel
R=$1
ncu -i $R --page details --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
want=('Duration','DRAM Throughput','Compute (SM) Throughput','Issue Slots Busy','Achieved Occupancy','Registers Per Thread','Executed Ipc Active','L2 Hit Rate','Warp Cycles Per Issued Instruction','Theoretical Occupancy','SM Frequency')
seen=set()
for r in rows[1:]:
    n=r[h.index('Metric Name')]
    if n in want and n not in seen:
        seen.add(n); print(f'{n:40s} {r[h.index(\"Metric Value\")]} {r[h.index(\"Metric Unit\")]}')
"
ncu -i $R --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
st=[]
for i,n in enumerate(h):
    if n.startswith('smsp__pcsamp_warps_issue_stalled') and not n.endswith('not_issued'):
        try: st.append((float(v[i].replace(',','')), n.replace('smsp__pcsamp_warps_issue_stalled_','')))
        except: pass
tot=sum(x for x,_ in st) or 1
print('stalls:', ', '.join(f'{n} {100*x/tot:.0f}%' for x,n in sorted(st,reverse=True)[:8]))
for i,n in enumerate(h):
    if n in ('smsp__inst_executed.sum','dram__bytes_read.sum','dram__bytes_write.sum'): print(n, v[i])
"
