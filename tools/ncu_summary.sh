#!/bin/bash
# tools/ncu_summary.sh <report.ncu-rep> [top]: key metrics + per-instruction stall summary
rep=$1; top=${2:-10}
ncu -i $rep --page details --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]
want=('Duration','DRAM Throughput','Issue Slots Busy','Executed Ipc Active','Achieved Active Warps Per SM','Executed Instructions','Registers Per Thread','L2 Hit Rate','Block Limit Shared Mem','Block Limit Registers')
for row in r[1:]:
    d=dict(zip(h,row))
    if d.get('Metric Name') in want: print('  ', d['Metric Name'], d['Metric Value'], d['Metric Unit'])
"
ncu -i $rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
r=list(csv.reader(sys.stdin)); h=r[0]; v=r[2]
d=dict(zip(h,v))
try:
    rd=float(d['dram__bytes_read.sum']); wr=float(d['dram__bytes_write.sum'])
    print('   dram read', rd, r[1][h.index('dram__bytes_read.sum')], 'write', wr, r[1][h.index('dram__bytes_write.sum')])
except Exception as e: print(e)
"
ncu -i $rep --page source --csv --print-source sass > /tmp/_sass.csv 2>/dev/null
python $(dirname $0)/sass_summary.py /tmp/_sass.csv $top
