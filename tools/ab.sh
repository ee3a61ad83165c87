#!/bin/bash
# Same-box A/B of DUALMESH_GATHER_CFG values on one config: alternating runs,
# element-loop CUDA-event times (tools/profile_step.py), then a bitwise check.
# usage: tools/ab.sh CONFIG "cfgA cfgB ..." [reps] [outfile]
conf=$1; cfgs=$2; reps=${3:-3}; out=${4:-gpurun_out/ab.log}
for r in $(seq $reps); do
  for cfg in $cfgs; do
    DUALMESH_GATHER_CFG=$cfg python tools/profile_step.py --config $conf --steps 8 | tail -4 | \
      python -c "import sys,json; r=[json.loads(l) for l in sys.stdin]; print('$conf cfg $cfg', 'elem %.4f'%(sum(x['elem_ms'] for x in r)/len(r)), 'total %.4f'%(sum(x['total_ms'] for x in r)/len(r)))" >> $out
  done
done
for cfg in $cfgs; do
  [ "$cfg" != "0" ] && python tools/cmp_cfg.py --config $conf --cfg $cfg >> $out
done
