#!/bin/bash
# symmetric scheme: seed stride sweep (C5 axis A shape)
for ss in 4 8 16; do echo "SS=$ss"; GGM_SEED_STRIDE=$ss timeout 200 python tools/sym_probe.py 2>&1 | grep "sym=1"; done
