#!/bin/bash
# symmetric vs plain scheme under the BK2 debug modes (0 normal, 1 TMEM loads only, 2 no epilogue)
for d in 0 1 2; do GGM_DEBUG_EPI=$d timeout 200 python tools/sym_probe.py 2>&1; done
