#!/bin/bash
# quick bench lines: tools/quick_bench.sh <config> [extra bench args]
cfg=$1; shift
timeout 600 python bench.py --config $cfg --steps 500 --warmup 10 --no-cpu-baseline "$@" 2>&1 | tail -1 | python -c "
import json,sys
t=sys.stdin.read()
try:
    d=json.loads(t)
except Exception:
    print('BENCH FAILED', t[-2000:]); sys.exit()
r=d['roofline']
print(d['config']['workload'], 'GFLOP/s=%.1f'%d['value'], 'ms=%.4f'%d['ms_per_step'], 'kern_ms=%.4f'%r['kernel_avg_ms'], 'frac=%.3f'%r['frac'], 'GBps=%.0f'%r['achieved'], d['stats_rank0'], 'clk', d['clocks'].get('sm_mhz'), 'part_ms', d.get('partition_ms'), d.get('partition_phase_ms'), d.get('layout_build_ms'), 'ktimes', d.get('kernel_times_us'))
"
