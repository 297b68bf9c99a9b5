#!/bin/bash
# usage: tools/phases.sh <config> <steps> [ENV=VAL ...]  -> compact phase table from bench.py
cfg=$1; steps=$2; shift 2
env "$@" python bench.py --config $cfg --steps $steps --warmup 2 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read().strip().splitlines()[-1])
print('$cfg $*', 'ms/step %.2f'%d['ms_per_step'], 'Gnnz/s %.2f'%(d['value']/1e9), 'fit %.6f'%d['fit_last'], 'clk', d['clocks']['sm_mhz'])
print('   ' + '  '.join('%s=%.2f'%(k, v['ms_per_launch']) for k,v in d['phases'].items() if v['ms_per_launch']>0.01))
"
