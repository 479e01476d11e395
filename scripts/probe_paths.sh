#!/bin/bash
# compare sweep paths: register loads vs TMA pipeline with 1 or 2 teams
for cfg in "reg 1" "tma 1" "tma 2"; do
  set -- $cfg
  echo "=== LRQ_SWEEP_PATH=$1 LRQ_TMA_TEAMS=$2"
  LRQ_SWEEP_PATH=$1 LRQ_TMA_TEAMS=$2 timeout 120 python scripts/probe_perf.py 32,10,fp32 33,3,fp64 28,3,fp64 | grep -E "wall|^   [PMFRZ] " | head -40
done
