#!/bin/bash
# Same-box A/B of environment settings on one config (element-loop CUDA events).
# usage: tools/ab_env.sh CONFIG reps outfile "ENV=.. ENV2=.." "ENV=.." ...
conf=$1; reps=$2; out=$3; shift 3
for r in $(seq $reps); do
  for envs in "$@"; do
    env $envs python tools/profile_step.py --config $conf --steps 8 | tail -4 | \
      python -c "import sys,json; r=[json.loads(l) for l in sys.stdin]; print('$conf [$envs]', 'elem %.4f'%(sum(x['elem_ms'] for x in r)/len(r)), 'bnd %.4f'%(sum(x['bnd_ms'] for x in r)/len(r)), 'vol %.4f'%(sum(x['vol_ms'] for x in r)/len(r)), 'total %.4f'%(sum(x['total_ms'] for x in r)/len(r)))" >> $out
  done
done
