#!/bin/bash
# Timing decomposition of BK2: normal / TMEM-loads-only / no-epilogue, for both kernel variants.
for pair in 1 0; do
  for dbg in 0 1 2; do
    echo "GGM_PAIR=$pair GGM_DEBUG_EPI=$dbg"
    GGM_PAIR=$pair GGM_DEBUG_EPI=$dbg timeout 120 python tools/perf_probe.py --sparse-only 2>&1 | grep "n=200000\|n=1000000"
  done
done
