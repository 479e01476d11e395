#!/bin/bash
# which (precision, group, kind) fails or wins on the 2-team TMA path
for tok in c64AF c64AR c64H4M c64H4F c64HF c128AF c128AR c128HM c128HF; do
  for teams in 1 2; do
    printf "%-8s teams=%s " $tok $teams
    if [[ $tok == c128* ]]; then cfg="25,3,fp64"; else cfg="32,4,fp32"; fi
    LRQ_SWEEP_PATH=$tok LRQ_TMA_TEAMS=$teams timeout 60 python scripts/probe_perf.py $cfg 2>&1 | grep -E "wall|Error" | tr '\n' ' '
    echo
  done
done
