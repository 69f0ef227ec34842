#!/bin/bash
# Same-session A/B: default libggm.so vs tools/variants/$1.so (alternating, twice).
for i in 1 2; do
  timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000" | sed "s/^/[base] /" | cut -c1-110
  GGM_LIB_PATH=tools/variants/$1.so timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000" | sed "s/^/[$1] /" | cut -c1-110
done
