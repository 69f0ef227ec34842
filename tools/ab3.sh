# Same-session A/B/C: default libggm.so vs two variants (alternating, twice).
for i in 1 2; do
  timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000 k=100 sym=1" | sed "s/^/[base] /" | cut -c1-100
  for v in "$@"; do
    GGM_LIB_PATH=tools/variants/$v.so timeout 120 python tools/sym_probe.py 2>&1 | grep "n=1000000 k=100 sym=1" | sed "s/^/[$v] /" | cut -c1-100
  done
done
