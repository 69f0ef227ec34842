#!/bin/bash
# symmetric scheme: seed sample fraction sweep (C5 axis A shape)
for ss in 32 64 128; do echo "SS=$ss"; GGM_SEED_FRAC=$ss timeout 200 python tools/sym_probe.py 2>&1 | grep "sym=1"; done
