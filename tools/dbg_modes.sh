for m in 0 2 3; do GGM_DEBUG_EPI=$m GGM_LIB_PATH=tools/variants/epidbg.so timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000 k=100 sym=1" | cut -c1-110; done
timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000 k=100 sym=1" | sed 's/^/[base] /' | cut -c1-110
