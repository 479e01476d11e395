#!/bin/bash
for k in "mid_sizes" "small_cases" "cfg1 or n14" "max_cut or cut_" "triangle"; do
  printf "%-20s " "$k"
  python -m pytest tests/test_gpu_parity.py -q -x -k "($k) or paths_agree" 2>&1 | tail -n 1
done
