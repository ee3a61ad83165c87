#!/bin/bash
# GPU sweep of the GATHER kernel shapes (DUALMESH_GATHER_CFG) and variants.
out=${1:-gpurun_out/sweep.log}
: > $out
for cfg in 0 1; do
  for conf in C5 C3; do
    DUALMESH_GATHER_CFG=$cfg python tools/profile_step.py --config $conf --steps 3 | tail -1 | sed "s/^/cfg$cfg /" >> $out
  done
done
for conf in C5 C3; do
  python tools/profile_step.py --config $conf --variant faces --steps 3 | tail -1 >> $out
  python tools/profile_step.py --config $conf --variant exact --steps 3 | tail -1 >> $out
  python tools/profile_step.py --config $conf --algo traditional --steps 3 | tail -1 >> $out
done
