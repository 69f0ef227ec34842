#!/bin/bash
for d in 0 3; do GGM_DEBUG_EPI=$d timeout 200 python tools/sym_probe.py 2>&1; done
