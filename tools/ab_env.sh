#!/bin/bash
# A/B of an env toggle in one GPU session (alternating, to cancel clock drift). Usage: ab_env.sh VAR=val
for i in 1 2; do
  timeout 300 python tools/sym_probe.py 2>&1 | grep "n=1000000" | sed "s/^/[base] /"
  env "$1" timeout 300 python tools/sym_probe.py 2>&1 | grep "n=1000000" | sed "s/^/[$1] /"
done
