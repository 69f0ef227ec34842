#!/bin/bash
# Timing decomposition of BK2 (plain scheme): normal / TMEM-loads-only / no-epilogue / no-threshold-work
./tools/tmem_bench
for dbg in 0 1 2 4; do
  echo "GGM_DEBUG_EPI=$dbg"
  GGM_DEBUG_EPI=$dbg timeout 120 python tools/perf_probe.py --sparse-only 2>&1 | grep "n=200000\|n=1000000"
done
