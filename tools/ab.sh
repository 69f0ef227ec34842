#!/bin/bash
# A/B: default build vs the 12-warp (384-thread) build, plain and symmetric
for i in 1 2; do
  timeout 200 python tools/sym_probe.py 2>&1 | sed 's/^/[320] /'
  cp paper_2407_19892_b200/libggm.so /tmp/libggm_320.so
  cp tools/libggm_384.so paper_2407_19892_b200/libggm.so
  timeout 200 python tools/sym_probe.py 2>&1 | sed 's/^/[384] /'
  cp /tmp/libggm_320.so paper_2407_19892_b200/libggm.so
done
